mkdir -p gpurun_out/r2e
timeout 300 python scripts/probe_perf.py c0 c1 > gpurun_out/r2e/graphs_on.jsonl 2> gpurun_out/r2e/on.err
HYLU_OPTIONS=graphs=0 timeout 300 python scripts/probe_perf.py c0 c1 > gpurun_out/r2e/graphs_off.jsonl 2> gpurun_out/r2e/off.err
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2e/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/gputests.log
