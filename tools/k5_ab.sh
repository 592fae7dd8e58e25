#!/bin/bash
# A/B timing of K5 contraction variants on config 4: default lib, then each variant lib
cd "$(dirname "$0")/.."
python tools/k5_time.py configs/cfg4_large.cfg 5 2>&1 | grep -v "^setup"
for v in "$@"; do
  echo "== $v"
  TG_LIB_VARIANT=paper_2511_20432_b200/_lib/variants/lib_$v.so python tools/k5_time.py configs/cfg4_large.cfg 5 2>&1 | grep -v "^setup"
done
