python -m pytest tests/test_gpu_kernels.py tests/test_gpu_projection.py tests/test_gpu_configs.py -x -q -k "not full_resolution" 2>&1 | tail -3
python - <<'PY'
import time, torch, sys
sys.path.insert(0, '.')
from paper_2502_11618_b200 import PointCloud, build_grid
from paper_2502_11618_b200.scenes import multi_station_hall
for n in (20_000_000, 100_000_000):
    pos, col, _ = multi_station_hall(n, device="cuda")
    c = PointCloud(pos, col); c.device_arrays(); torch.cuda.synchronize()
    for rep in range(2):
        t = time.perf_counter(); g = build_grid(c, 1.0); g.scene(); torch.cuda.synchronize()
        print(n, "build_grid + Morton scene", f"{(time.perf_counter() - t) * 1e3:.1f} ms")
PY
