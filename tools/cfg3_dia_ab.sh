#!/bin/bash
cd "$(dirname "$0")/.."
python tools/k2_step_rate.py configs/cfg3_contour_hatch.cfg 5 | cut -c1-200
for v in "$@"; do echo "== $v"; TG_LIB_VARIANT=paper_2511_20432_b200/_lib/variants/lib_$v.so python tools/k2_step_rate.py configs/cfg3_contour_hatch.cfg 5 | cut -c1-200; done
