D=gpurun_out/r2ai; mkdir -p $D
for rep in 1 2; do
for v in base i2p4 i2p8 p16 ch32 p16ch32; do
    L=""; C=64
    case $v in i2p4|i2p8|p16) L=variants/$v.so;; ch32) C=32;; p16ch32) L=variants/p16.so; C=32;; esac
    HYLU_HUB_CHUNK=$C HYLU_LIB_PATH=$L K=8 timeout 300 python scripts/batch_time.py | sed "s/^/{\"v\": \"$v\", \"r\": /; s/\$/}/" >> $D/t.jsonl 2>> $D/err.txt
done
done
