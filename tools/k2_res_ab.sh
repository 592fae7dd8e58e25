#!/bin/bash
# K2 resident (shared-memory) solve vs the streaming single-sweep solve on small grids
cd "$(dirname "$0")/.."
for c in configs/cfg2_raster_layer.cfg configs/cfg0_parity.cfg; do
  echo -n "resident  "; python tools/k2_step_rate.py $c 5 | cut -c1-170
  echo -n "streaming "; TG_K2_NO_RESIDENT=1 python tools/k2_step_rate.py $c 5 | cut -c1-170
done
