mkdir -p gpurun_out/r2d
for v in r1 cur r1 cur; do HYLU_LIB_PATH=variants/$v.so timeout 300 python scripts/batch_time.py >> gpurun_out/r2d/t.jsonl 2>> gpurun_out/r2d/t.err; done
for v in r1 cur; do HYLU_LIB_PATH=variants/$v.so K=1 timeout 600 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d/launch_$v.csv python scripts/batch_time.py > /dev/null 2>&1; done
