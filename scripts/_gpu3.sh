mkdir -p gpurun_out/r2c
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/r2c/smi.txt
for v in r1 cur r1 cur; do HYLU_LIB_PATH=variants/$v.so timeout 300 python scripts/batch_time.py >> gpurun_out/r2c/t.jsonl 2>> gpurun_out/r2c/t.err; done
