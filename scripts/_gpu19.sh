D=gpurun_out/r2t; mkdir -p $D
timeout 2400 python -m pytest tests -m gpu -q > $D/gputests.log 2>&1; echo "tests rc=$?" >> $D/gputests.log
timeout 1800 python bench.py --steps 10 --warmup 3 > $D/bench.out 2> $D/bench.err; echo "bench rc=$?" >> $D/bench.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for c in c0 c1 c2; do
  python scripts/single_step.py $c solve > $D/plain_$c.log 2>&1 && timeout 900 /usr/local/cuda/bin/ncu --metrics $M --clock-control none --csv --log-file $D/kr_$c.csv python scripts/single_step.py $c solve > /dev/null 2>&1
done
python scripts/batch_step.py 4096 1 > $D/plain_c4.log 2>&1 && timeout 900 /usr/local/cuda/bin/ncu --metrics $M --clock-control none --csv --log-file $D/kr_c4.csv python scripts/batch_step.py 4096 1 > /dev/null 2>&1
python scripts/single_step.py c3k48 > $D/plain_c3.log 2>&1 && timeout 1500 /usr/local/cuda/bin/ncu --metrics $M --clock-control none --csv --log-file $D/kr_c3.csv python scripts/single_step.py c3k48 > /dev/null 2>&1
ls -la $D
