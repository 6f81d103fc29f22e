python -m pytest tests/test_gpu_projection.py tests/test_gpu_configs.py -x -q -k "not full_resolution and not c4" 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['stages_ms'], d['roofline']['other']['frac'])"; done
