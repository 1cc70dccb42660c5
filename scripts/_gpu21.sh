D=gpurun_out/r2w; mkdir -p $D
for rep in 1 2; do
for v in ws12 ws12c128 ws12c160 ws8c160 ws14; do
    L=""; O=""
    case $v in ws12) O="pipe_ws=12";; ws12c128) O="pipe_ws=12"; L=variants/c128.so;; ws12c160) O="pipe_ws=12"; L=variants/c160.so;; ws8c160) O="pipe_ws=8"; L=variants/c160.so;; ws14) O="pipe_ws=14";; esac
    HYLU_OPTIONS=$O HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
