set -x
D=gpurun_out/r2f; mkdir -p $D
nproc > $D/nproc.txt; lscpu | head -20 >> $D/nproc.txt
timeout 2400 python -m pytest tests -m gpu -x -q --durations=30 > $D/gputests.log 2>&1; echo "tests rc=$?" >> $D/gputests.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $D/bench.out 2> $D/bench.err; echo "bench rc=$?" >> $D/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $D/bench_ref.out 2> $D/bench_ref.err; echo "rc=$?" >> $D/bench_ref.err
