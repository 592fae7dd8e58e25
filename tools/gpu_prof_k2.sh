set -x
python tools/profile_sim.py configs/cfg4_large.cfg 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${K2_KERNEL:-k2_cg1_kernel} -s 1 -c 1 -o gpurun_out/k2_full python tools/profile_sim.py configs/cfg4_large.cfg 2 > gpurun_out/ncu_k2.log 2>&1; echo ncu=$?
cat gpurun_out/prof_plain.log
