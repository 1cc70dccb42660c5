D=gpurun_out/r2r; mkdir -p $D
for rep in 1 2; do
for v in default pf16 pf64 pf1k; do
    if [ $v = default ]; then L=""; else L=variants/$v.so; fi
    HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
