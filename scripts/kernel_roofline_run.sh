#!/bin/bash
# One ncu metric pass over every launch of c0, c1, c2 (factorize + solve), c4 (one batched
# refactorize+solve pass over 4096 instances) and c3 (factorize); CSVs into gpurun_out/.
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
mkdir -p gpurun_out
for c in c0 c1 c2; do
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/kr_$c.csv python scripts/single_step.py $c solve > /dev/null 2>&1
done
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/kr_c4.csv python scripts/batch_step.py 4096 1 > /dev/null 2>&1
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/kr_c3.csv python scripts/single_step.py c3k48 > /dev/null 2>&1
ls -la gpurun_out/kr_*.csv
