D=gpurun_out/r2am; mkdir -p $D
python -m pytest tests -m gpu -x -q -k "solve_multi" > $D/tests.log 2>&1; echo "rc=$?" >> $D/tests.log
timeout 1500 python scripts/multi_rhs_probe.py c0 c1 c2 c3k32 > $D/t.jsonl 2> $D/err.txt
