D=gpurun_out/r2j; mkdir -p $D
for rep in 1 2; do
for v in default p8 p6 p8m3 p2; do
    if [ $v = default ]; then L=""; else L=variants/$v.so; fi
    HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/p2w.jsonl 2>> $D/err.txt
done
done
