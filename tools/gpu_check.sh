set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
python bench.py --steps 2 --warmup 1 --ncu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --ncu > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_partial -s 1 -c 1 -o gpurun_out/k1_full python bench.py --steps 2 --warmup 1 --ncu > gpurun_out/ncu2.log 2>&1; echo ncu=$?
tail -3 gpurun_out/pytest_gpu.log
cat gpurun_out/bench.log | tail -2
