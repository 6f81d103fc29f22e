python -m pytest tests/test_gpu_unet.py tests/test_gpu_engine.py -x -q 2>&1 | tail -1
for a in 0 1; do for r in 1 2; do echo "l2hints=$a $(LS_UNET_L2HINTS=$a python scripts/time_unet.py | tail -1)"; done; done
for a in 0 1; do LS_UNET_L2HINTS=$a python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench l2hints=$a', round(d['value'],1), round(d['stages_ms']['unet']*1e3,1))"; done
