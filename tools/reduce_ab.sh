#!/bin/bash
# Per-iteration solve time with the batched partial-sum read (default build)
# against a saved build (variants/old.so), configs 2 (resident), 4 (streaming),
# 3 (CSR/DIA), alternated twice on the same box.
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for c in configs/cfg2_raster_layer.cfg configs/cfg4_large.cfg configs/cfg3_contour_hatch.cfg; do
    n=200; [ $c = configs/cfg3_contour_hatch.cfg ] && n=100
    TG_LIB_VARIANT=$PWD/variants/old.so python tools/k2_iter_time.py $c $n
    python tools/k2_iter_time.py $c $n
  done
done
