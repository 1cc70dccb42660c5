D=gpurun_out/r2ar; mkdir -p $D
for rep in 1 2; do
for v in base m4k16 m4 k16; do
  L=""; [ $v != base ] && L=variants/$v.so
  HYLU_LIB_PATH=$L timeout 900 python scripts/probe_perf.py c2 c3 --c3k 32 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
