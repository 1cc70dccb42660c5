D=gpurun_out/r2i; mkdir -p $D
for rep in 1 2; do
for v in default hp4 hp16 hp32; do
  for ch in 64 32 16; do
    if [ $v = default ]; then L=""; else L=variants/$v.so; fi
    HYLU_LIB_PATH=$L HYLU_HUB_CHUNK=$ch K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"chunk\": $ch, \"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/hub.jsonl 2>> $D/err.txt
  done
done
done
