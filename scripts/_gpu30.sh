D=gpurun_out/r2al; mkdir -p $D
HYLU_LIB_PATH=variants/bulkx.so python -m pytest tests -m gpu -x -q -k "kernel_override or factorize_matches or c3_intermediate or golden or maps" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in old bulkx; do
  L=variants/$v.so
  HYLU_LIB_PATH=$L timeout 900 python scripts/probe_perf.py c2 c3 --c3k 32 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
