# round-2 checkpoint 3: full GPU suite, smoke, default bench x2, 20M / C1 lines, reference arm
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite3.log 2>&1; tail -2 gpurun_out/r02_gpu_suite3.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_100m_v3_$i.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r02_bench_100m_v3_$i.json').read().strip().splitlines()[-1]); print('100M', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), round(d['roofline']['frac'],3), round(d['roofline']['other']['frac'],3), d['parity']['bit_exact'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
python bench.py --steps 20 --warmup 5 --points 20000000 --no-cpu-baseline > gpurun_out/r02_bench_20m_v3.json 2>/dev/null; tail -c 200 gpurun_out/r02_bench_20m_v3.json
python bench.py --steps 200 --warmup 10 --points 1000000 --width 512 --height 512 --unet reduced > gpurun_out/r02_bench_c1_v3.json 2>/dev/null; tail -c 200 gpurun_out/r02_bench_c1_v3.json
