timeout 900 python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -2
for r in 1 2; do echo "fused $(timeout 120 python scripts/time_unet.py | tail -1)"; echo "unfused $(LS_UNET_UPFUSE=0 timeout 120 python scripts/time_unet.py | tail -1)"; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__cycles_active.avg,smsp__cycles_active.avg
N=1 timeout 300 ncu --metrics $M --clock-control none -k regex:k_conv -c 21 --csv python scripts/time_unet.py > gpurun_out/m_upfuse.csv 2>/dev/null
