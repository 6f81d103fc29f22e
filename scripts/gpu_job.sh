python -m pytest tests/test_gpu_unet.py tests/test_gpu_bridge.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
python -m pytest tests/test_gpu_configs.py -x -q -k full_resolution -s 2>&1 | grep -E "DEFAULT|passed|failed"
for r in 1 2; do python scripts/time_unet.py | tail -1; done
