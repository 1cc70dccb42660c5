D=gpurun_out/r2ab; mkdir -p $D

for rep in 1 2; do
for v in ws6 c192ws4 c192ws6 c256ws4; do
    L=""; O=""
    case $v in ws6) O="pipe_ws=6";; c192ws4) O="pipe_ws=4"; L=variants/c192.so;; c192ws6) O="pipe_ws=6"; L=variants/c192.so;; c256ws4) O="pipe_ws=4"; L=variants/c256.so;; esac
    HYLU_OPTIONS=$O HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
