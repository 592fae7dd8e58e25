python tools/k2_iter_time.py configs/cfg2_raster_layer.cfg 200
python tools/k2_iter_time.py configs/cfg0_parity.cfg 200
TG_LIB_VARIANT=$PWD/variants/old.so python tools/k2_iter_time.py configs/cfg0_parity.cfg 200
bash tools/gpu_full.sh
