D=gpurun_out/final6; mkdir -p $D
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > $D/gputests.txt
python bench.py > $D/bench.json 2> $D/bench.err
python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > $D/smoke.txt 2>&1
tail -3 $D/gputests.txt; tail -c 300 $D/bench.json; tail -2 $D/smoke.txt
