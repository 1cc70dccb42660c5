D=gpurun_out/r2ah; mkdir -p $D
K=1 python scripts/batch_time.py > $D/plain.log 2>&1 && \
K=1 timeout 1500 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_bt_hub -s 7 -c 1 -o $D/hub python scripts/batch_time.py > $D/ncu.log 2>&1; echo "rc=$?" >> $D/ncu.log
