for r in 1 2 3; do echo "new $(timeout 120 python scripts/time_unet.py | tail -1)"; echo "old $(LS_LIB_PATH=scripts/exp/liblidarsplat_old.so timeout 120 python scripts/time_unet.py | tail -1)"; done
