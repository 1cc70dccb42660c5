D=gpurun_out/r2h; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q -k "solve_multi" > $D/new.log 2>&1; echo "rc=$?" >> $D/new.log
