timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_configs.py -x -q -k "not c4 and not c5" 2>&1 | tail -1
for r in 1 2; do echo "by-input $(timeout 120 python scripts/time_unet.py | tail -1)"; echo "kx2 $(LS_CONV_PX64=0 timeout 120 python scripts/time_unet.py | tail -1)"; done
