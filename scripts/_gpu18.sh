D=gpurun_out/r2s; mkdir -p $D
timeout 900 python -m pytest tests -m gpu -x -q -k "kernel_override or factorize_matches or golden or refactorize or full_size_factor or solve_multi or cli" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in off auto on; do
  if [ $v = off ]; then O="fanin_mega=0"; elif [ $v = on ]; then O="fanin_mega=1"; else O=""; fi
  HYLU_OPTIONS=$O timeout 900 python scripts/probe_perf.py c0 c1 c2 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
