D=gpurun_out/r2ag; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q > $D/gputests.log 2>&1; echo "tests rc=$?" >> $D/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "rc=$?" >> $D/smoke.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $D/bench.out 2> $D/bench.err; echo "bench rc=$?" >> $D/bench.err

