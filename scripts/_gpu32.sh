D=gpurun_out/r2ap; mkdir -p $D

for rep in 1 2; do
for v in pdl nopdl; do
  O=""; [ $v = nopdl ] && O="pdl=0"
  HYLU_OPTIONS=$O timeout 900 python scripts/probe_perf.py c0 c1 c2 c3 --c3k 32 | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
