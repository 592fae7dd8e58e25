# round-2 profile set: config-4 step launch list + full captures of the K5
# contraction and the K2 solve, and the config-1 bench launch list
set -x
python tools/k5_prof.py > gpurun_out/p_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/r02b_launches_cfg4_step.csv python tools/k5_prof.py > gpurun_out/p_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sf_contract_kernel -s 1 -c 1 \
    -o gpurun_out/r02b_k5_contract python tools/k5_prof.py > gpurun_out/p_k5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2_cg1_kernel -c 1 \
    -o gpurun_out/r02b_k2_cg1 python tools/k5_prof.py > gpurun_out/p_k2.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --theta-steps 0 --theta-sharded 0 > gpurun_out/p_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02b_launches_bench.csv python bench.py --steps 2 --warmup 3 --ncu \
    --no-cpu-baseline --theta-steps 0 --theta-sharded 0 > gpurun_out/p_bn.log 2>&1
ls -la gpurun_out | tail -12
