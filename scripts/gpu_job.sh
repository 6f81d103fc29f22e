# GPU-box job used for the round-2 final validation (run via gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/gpu_job.sh'
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_suite_final4.log 2>&1; tail -2 gpurun_out/r02_gpu_suite_final4.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_bench_100m_final4_$i.json 2>/dev/null; done
python bench.py --steps 200 --warmup 10 --points 1000000 --width 512 --height 512 --unet reduced > gpurun_out/r02_bench_c1_final4.json 2>/dev/null
python bench.py --steps 20 --warmup 5 --points 20000000 --no-cpu-baseline > gpurun_out/r02_bench_20m_final4.json 2>/dev/null
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02_ref_final4.json 2>/dev/null
timeout 600 python scripts/c5_views.py > gpurun_out/r02_c5_views_final4.jsonl 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:^k_ -c 200 --csv --log-file gpurun_out/r02_bench_launches_final4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_conv -c 21 --csv --log-file gpurun_out/r02_unet_layers_final4.csv python scripts/time_unet.py > /dev/null 2>&1
