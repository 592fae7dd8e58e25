#!/bin/bash
cd "$(dirname "$0")/.."
c=configs/cfg4_large.cfg
for rep in 1 2; do
  echo -n "strip   "; python tools/k2_step_rate.py $c 3 | cut -c1-150
  echo -n "nostrip "; TG_K2_NO_STRIP=1 python tools/k2_step_rate.py $c 3 | cut -c1-150
done
tools/k2_res_ab.sh
