D=gpurun_out/r2ae; mkdir -p $D

for rep in 1 2; do
for v in sk1 sk2 sk3 sk4; do
    L=""; O=""
    O="pipe_skew=${v#sk}"
    HYLU_OPTIONS=$O HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
