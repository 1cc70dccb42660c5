D=gpurun_out/r2m; mkdir -p $D
T=${1:-racecheck}
python scripts/sanitize_probe.py > $D/plain_$T.log 2>&1 && \
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool $T $([ $T = racecheck ] && echo --racecheck-report analysis) python scripts/sanitize_probe.py > $D/$T.log 2>&1; echo "rc=$?" >> $D/$T.log
