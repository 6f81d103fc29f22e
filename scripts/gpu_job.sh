# round-2 checkpoint: full GPU suite, default bench (100M), C1/C2 configs, reference arm, ncu launch list
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite.log 2>&1; tail -3 gpurun_out/r02_gpu_suite.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_100m.json 2> gpurun_out/r02_bench_100m.err; tail -c 600 gpurun_out/r02_bench_100m.json
python bench.py --steps 20 --warmup 5 --points 20000000 --no-cpu-baseline > gpurun_out/r02_bench_20m.json 2>&1
python bench.py --steps 200 --warmup 10 --points 1000000 --width 512 --height 512 --unet reduced > gpurun_out/r02_bench_c1.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_reference_100m.json 2>&1; tail -c 400 gpurun_out/r02_reference_100m.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02_bench_ncu.log 2>&1; tail -2 gpurun_out/r02_bench_ncu.log
