python -m pytest tests/test_gpu_projection.py -x -q 2>&1 | tail -1
for v in base nohint base nohint; do
  if [ $v = base ]; then unset LS_LIB_PATH; else export LS_LIB_PATH=scripts/exp/liblidarsplat_$v.so; fi
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['stages_ms']; print('$v', round(d['value'],1), {k: round(v*1e3,1) for k,v in s.items()})"
done
unset LS_LIB_PATH; python scripts/time_unet.py | tail -1
