timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
python tools/k2_trace.py
python tools/k2_trace.py configs/cfg2_raster_layer.cfg
