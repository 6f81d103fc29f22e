timeout 900 python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -1
for r in 1 2; do echo "$(timeout 120 python scripts/time_unet.py | tail -1)"; done
