D=gpurun_out/r2aq; mkdir -p $D
python -m pytest tests -m gpu -x -q -k "solve or batched or golden or refine" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in pdl nopdl; do
  O=""; [ $v = nopdl ] && O="pdl=0"
  HYLU_OPTIONS=$O timeout 900 python scripts/probe_perf.py c0 c1 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
  HYLU_OPTIONS=$O K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"c4\": /; s/\$/}/" >> $D/t4.jsonl 2>> $D/err.txt
done
done
