python -m pytest tests/test_gpu_engine.py -x -q 2>&1 | tail -2
for g in 0 1; do
python bench.py --steps 200 --warmup 10 --points 1000000 --width 512 --height 512 --unet reduced --no-cpu-baseline --graph $g 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C1 graph=$g', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), d['frame_ms'])"
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --graph $g 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3 graph=$g', round(d['value'],1), 'e2e', round(d['e2e']['value'],1))"
done
