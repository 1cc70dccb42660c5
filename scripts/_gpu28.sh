D=gpurun_out/r2aj; mkdir -p $D
python -m pytest tests -m gpu -x -q -k "kernel_override or factorize_matches or golden or refactorize or swap or perturb or Breakdown" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in old new; do
  if [ $v = new ]; then L=""; else L=variants/$v.so; fi
  HYLU_LIB_PATH=$L timeout 900 python scripts/probe_perf.py c0 c1 c2 c3 --c3k 32 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
