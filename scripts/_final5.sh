D=gpurun_out/final5; mkdir -p $D
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $D/gputests.txt
python bench.py > $D/bench.json 2> $D/bench.err
python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for c in c0 c1; do timeout 600 ncu --metrics $M --clock-control none --csv --log-file $D/kr_$c.csv python scripts/single_step.py $c solve > /dev/null 2>&1; done
tail -3 $D/gputests.txt; tail -c 200 $D/bench.json; tail -2 $D/smoke.txt
