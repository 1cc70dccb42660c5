D=gpurun_out/r2g; mkdir -p $D
timeout 1500 python -m pytest tests -m gpu -x -q -k "refine or kernel_override or batched or factorize_matches" > $D/new.log 2>&1; echo "rc=$?" >> $D/new.log
timeout 2400 python -m pytest tests -m gpu -q > $D/gputests.log 2>&1; echo "tests rc=$?" >> $D/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.log 2>&1; echo "rc=$?" >> $D/smoke.log
