set -x
mkdir -p gpurun_out/r2a
nproc > gpurun_out/r2a/nproc.txt; lscpu | head -20 >> gpurun_out/r2a/nproc.txt
timeout 1800 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/r2a/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r2a/gputests.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool memcheck python scripts/sanitize_probe.py > gpurun_out/r2a/memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/memcheck.log
timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report analysis python scripts/sanitize_probe.py > gpurun_out/r2a/racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/racecheck.log
timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool synccheck python scripts/sanitize_probe.py > gpurun_out/r2a/synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r2a/synccheck.log
timeout 1800 python bench.py --steps 10 --warmup 3 > gpurun_out/r2a/bench.out 2> gpurun_out/r2a/bench.err; echo "bench rc=$?" >> gpurun_out/r2a/bench.err
