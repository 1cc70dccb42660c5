D=gpurun_out/r2n; mkdir -p $D
C=${1:-c3k48}
python scripts/single_step.py $C > $D/plain_$C.log 2>&1 && \
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fi_upd_kc --csv --log-file $D/kc_$C.csv python scripts/single_step.py $C > /dev/null 2>&1
IDX=$(python - "$D/kc_$C.csv" <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; KN=h.index("Kernel Name"); MV=h.index("Metric Value")
ts=[(float(r[MV].replace(",","")), r[KN]) for r in rows[1:]]
kc=[(i,t) for i,(t,n) in enumerate([(t,n) for t,n in ts if "k_fi_upd_kc(" in n])]
best=max(kc,key=lambda x:x[1]); print(best[0])
PY
)
echo "heaviest kc launch index $IDX" > $D/idx_$C.txt
timeout 1500 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:"k_fi_upd_kc$" -s $IDX -c 1 -o $D/kc_$C python scripts/single_step.py $C > $D/ncu_$C.log 2>&1; echo "rc=$?" >> $D/ncu_$C.log
