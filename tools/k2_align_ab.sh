#!/bin/bash
cd "$(dirname "$0")/.."
c=configs/cfg4_large.cfg
for rep in 1 2; do
  echo -n "aligned   "; python tools/k2_step_rate.py $c 3 | cut -c1-150
  echo -n "unaligned "; TG_K2_ALIGNED=0 python tools/k2_step_rate.py $c 3 | cut -c1-150
  echo -n "nostrip   "; TG_K2_NO_STRIP=1 python tools/k2_step_rate.py $c 3 | cut -c1-150
done
for a in 1 0; do
TG_K2_ALIGNED=$a ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k2_cg1_kernel -c 1 python tools/k5_prof.py 2>&1 | grep -E "dram__|gpu__time"
done
