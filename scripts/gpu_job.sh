timeout 900 python -m pytest tests/test_gpu_unet.py tests/test_gpu_configs.py tests/test_gpu_engine.py tests/test_gpu_bridge.py -x -q 2>&1 | tail -3
