set -x
python -m pytest tests/test_gpu_configs.py tests/test_gpu_shard.py tests/test_gpu_filter.py tests/test_gpu_engine.py tests/test_bench_contract.py -x -q > gpurun_out/r02_gpu_tests_4.log 2>&1; tail -15 gpurun_out/r02_gpu_tests_4.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_v1.json 2> gpurun_out/r02_bench_v1.err; tail -c 4000 gpurun_out/r02_bench_v1.json; tail -5 gpurun_out/r02_bench_v1.err
