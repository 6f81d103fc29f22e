LS_LIB_PATH=scripts/exp/liblidarsplat_g3.so timeout 600 python -m pytest tests/test_gpu_unet.py -x -q -k "layer" 2>&1 | tail -1
for r in 1 2; do for v in base g3 g1; do
 if [ $v = base ]; then L="X=1"; else L="LS_LIB_PATH=scripts/exp/liblidarsplat_$v.so"; fi
 echo "$v $(env $L timeout 120 python scripts/time_unet.py | tail -1)"
done; done
M=gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__cycles_active.avg,smsp__cycles_active.avg
LS_LIB_PATH=scripts/exp/liblidarsplat_g3.so N=1 timeout 300 ncu --metrics $M --clock-control none -k regex:k_conv -c 22 --csv python scripts/time_unet.py > gpurun_out/m_g3.csv 2>/dev/null
