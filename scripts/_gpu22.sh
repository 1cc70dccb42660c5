D=gpurun_out/r2z; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q -k "batched or sharded or golden" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in norinv new; do
    L=""; O=""
    case $v in norinv) L=variants/norinv.so;; esac
    HYLU_OPTIONS=$O HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
