mkdir -p gpurun_out/r2b
for v in 0 1 2 0 1 2; do HYLU_LIB_PATH=variants/acq$v.so timeout 300 python scripts/batch_time.py >> gpurun_out/r2b/acq.jsonl 2>> gpurun_out/r2b/acq.err; done
timeout 900 python scripts/lit_probe.py 16 > gpurun_out/r2b/lit16.jsonl 2> gpurun_out/r2b/lit16.err
timeout 600 python scripts/lit_probe.py 8 > gpurun_out/r2b/lit8.jsonl 2> gpurun_out/r2b/lit8.err
