python -m pytest tests/test_gpu_projection.py tests/test_gpu_configs.py tests/test_gpu_shard.py -x -q -k "not full_resolution and not c4" 2>&1 | tail -1
for r in 1 2 3; do python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print(round(d['value'],1), {k: round(v*1e3,1) for k,v in s.items()})"; done
