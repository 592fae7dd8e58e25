#!/bin/bash
# K2 per-iteration time with and without the strip tiles (config 4), strip weights
cd "$(dirname "$0")/.."
c=configs/cfg4_large.cfg
for rep in 1 2; do
  for w in 5 6 7; do echo -n "w=$w "; TG_K2_STRIP_W=$w python tools/k2_step_rate.py $c 3 | cut -c1-150; done
  echo -n "nostrip "; TG_K2_NO_STRIP=1 python tools/k2_step_rate.py $c 3 | cut -c1-150
done
