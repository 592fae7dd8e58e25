# round-2 (third set) profiles: config-4 step launch list, full captures of the
# K2 streaming solve with strip tiles (config 4) and of the resident solve (config 2)
cd "$(dirname "$0")/.."
set -x
python tools/k5_prof.py > gpurun_out/c_plain.log 2>&1 || exit 1
python tools/step_profile.py configs/cfg2_raster_layer.cfg 0 3 > gpurun_out/c_plain2.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02c_launches_cfg4_step.csv python tools/k5_prof.py > gpurun_out/c_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_cg1_kernel -c 1 \
    -o gpurun_out/r02c_k2_cg1_strip python tools/k5_prof.py > gpurun_out/c_k2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_res_kernel -s 2 -c 1 \
    -o gpurun_out/r02c_k2_res_cfg2 python tools/step_profile.py configs/cfg2_raster_layer.cfg 0 3 > gpurun_out/c_res.log 2>&1
ls -la gpurun_out | tail -8
