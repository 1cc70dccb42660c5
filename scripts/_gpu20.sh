D=gpurun_out/r2u; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q -k "batched or sharded or golden" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2 3; do
for v in old new; do
    if [ $v = new ]; then L=""; else L=variants/$v.so; fi
    HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
