for r in 1; do
echo "base $(timeout 120 python scripts/time_unet.py | tail -1)"
for mb in 16 32 48; do
h=$(python -c "print(round($mb/128,3))")
echo "sa$mb h$h $(LS_L2_SETASIDE_MB=$mb LS_UNET_L2WIN=$h timeout 120 python scripts/time_unet.py | tail -1)"
echo "sa$mb h1 $(LS_L2_SETASIDE_MB=$mb LS_UNET_L2WIN=1.0 timeout 120 python scripts/time_unet.py | tail -1)"
done
done
