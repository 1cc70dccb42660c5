D=gpurun_out/r2as; mkdir -p $D
HYLU_OPTIONS=pipe_groups=4 python -m pytest tests -m gpu -x -q -k "batched or sharded or golden" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
for rep in 1 2; do
for v in g2 g4 g4ws4 g4ws8; do
  case $v in g2) O="";; g4) O="pipe_groups=4";; g4ws4) O="pipe_groups=4,pipe_ws=4";; g4ws8) O="pipe_groups=4,pipe_ws=8";; esac
  HYLU_OPTIONS=$O K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
