python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -1
for a in 0 1 0 1; do echo "l2hints=$a $(LS_UNET_L2HINTS=$a python scripts/time_unet.py | tail -1)"; done
