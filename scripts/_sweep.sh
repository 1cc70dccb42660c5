out=gpurun_out/rowstage.txt; : > $out
python scripts/batch_time.py 2>&1 | tail -1 >> $out
HYLU_OPTIONS=pipe_order=0 python scripts/batch_time.py 2>&1 | tail -1 >> $out
python -m pytest tests/test_gpu_parity.py -q -x -k "launch_options or batched" 2>&1 | tail -3 >> $out
HYLU_LIB_PATH=variants/libhylu_trace.so python scripts/pipe_trace.py > gpurun_out/pipe_trace_lm.txt 2>&1
cat $out
