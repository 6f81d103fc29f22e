timeout 600 python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -1
LS_CONV_PAIR_SIDE=1 timeout 600 python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -1
LS_CONV_PAIR_SIDE=1 LS_CONV_PAIR=2 timeout 600 python -m pytest tests/test_gpu_unet.py -x -q -k "layer or bit_identical" 2>&1 | tail -1
for r in 1 2; do echo "auto $(timeout 120 python scripts/time_unet.py | tail -1)"; echo "stacked $(LS_CONV_PAIR_SIDE=0 timeout 120 python scripts/time_unet.py | tail -1)"; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__cycles_active.avg,smsp__cycles_active.avg
N=1 timeout 300 ncu --metrics $M --clock-control none -k regex:k_conv -c 22 --csv python scripts/time_unet.py > gpurun_out/m_side.csv 2>/dev/null
