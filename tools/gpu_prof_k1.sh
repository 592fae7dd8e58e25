set -x
python bench.py --steps 2 --warmup 1 --ncu --theta-steps 0 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_k1.csv python bench.py --steps 2 --warmup 1 --ncu --theta-steps 0 > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k1_partial -s 1 -c 1 -o gpurun_out/k1_full python bench.py --steps 2 --warmup 1 --ncu --theta-steps 0 > gpurun_out/ncu2.log 2>&1; echo ncu=$?
python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log
