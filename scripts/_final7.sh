D=gpurun_out/final7; mkdir -p $D
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $D/bench_launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --configs "" > $D/ncu_bench.log 2>&1
wc -l $D/bench_launches.csv; tail -c 300 $D/ncu_bench.log
python scripts/batch_time.py 2>&1 | tail -3
