python -m pytest tests/test_gpu_unet.py -x -q 2>&1 | tail -1
for v in split1 split2 split3; do for r in 1 2; do echo "$v $(LS_LIB_PATH=scripts/exp/liblidarsplat_$v.so python scripts/time_unet.py | tail -1)"; done; done
