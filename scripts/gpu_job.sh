# round-2 checkpoint 2: full GPU suite, default bench (100M), launch list, one --set full of the top kernels
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite2.log 2>&1; tail -2 gpurun_out/r02_gpu_suite2.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_100m_v2.json 2> gpurun_out/r02_bench_100m_v2.err; tail -c 300 gpurun_out/r02_bench_100m_v2.json
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_frame_launches_v2.csv python scripts/profile_frame.py --points 100000000 --frames 3 --unet default > /dev/null 2>&1; echo launches $?
ncu --set full --import-source on --clock-control none -k regex:"k_conv_px2|k_frame_pass" --launch-skip 6 --launch-count 6 -o gpurun_out/r02_top_full python scripts/profile_frame.py --points 100000000 --frames 3 --unet default > gpurun_out/r02_top_full.log 2>&1; echo full $?
