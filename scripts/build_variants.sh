#!/bin/bash
# Build kernel variants of libhylu_b200.so into variants/<name>.so (in parallel):
#   scripts/build_variants.sh name1 "-DFOO=1" name2 "-DFOO=2" ...
# then time each on the GPU with HYLU_LIB_PATH=variants/<name>.so.
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -ge 2 ]; do
  python -c "from paper_2509_07690_b200 import build as b; b.build_cuda(force=True, out='variants/$1.so', extra='$2')" &
  shift 2
done
wait
ls variants
