D=gpurun_out/final2; mkdir -p $D
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $D/gputests.txt
python bench.py > $D/bench.json 2> $D/bench.err
python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
python scripts/batch_step.py 4096 1 > $D/plain_c4.log 2>&1 && timeout 900 ncu --metrics $M --clock-control none --csv --log-file $D/kr_c4.csv python scripts/batch_step.py 4096 1 > /dev/null 2>&1
HYLU_LIB_PATH=variants/libhylu_trace.so python scripts/pipe_trace.py > $D/pipe_trace.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
tail -3 $D/gputests.txt; tail -c 300 $D/bench.json; tail -2 $D/smoke.txt
