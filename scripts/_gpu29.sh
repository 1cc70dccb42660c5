D=gpurun_out/r2ak; mkdir -p $D
python -m pytest tests -m gpu -x -q -k "kernel_override or factorize_matches or c2_full or c3_intermediate or golden or maps or refactorize" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in old new nobulk; do
  L=""; [ $v != new ] && L=variants/$v.so
  HYLU_LIB_PATH=$L timeout 900 python scripts/probe_perf.py c1 c2 c3 --c3k 32 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
