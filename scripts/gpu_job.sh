timeout 900 python -m pytest tests/test_gpu_unet.py -x -q -k "fused_up or bit_identical" 2>&1 | tail -2
