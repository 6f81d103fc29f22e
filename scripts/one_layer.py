"""Run one conv layer a few times (for ncu captures): python scripts/one_layer.py d0c1"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("LS_TIME_LAYER_NO_MAIN", "1")
from time_layer import layer, H, W  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "d0c1"
cfg = {"e0c1": dict(c0=8, c1=0, cout=32, h=H, w=W),
       "e0c2": dict(c0=32, c1=0, cout=32, h=H, w=W, pool=True),
       "d0c1": dict(c0=32, c1=32, cout=32, h=H, w=W),
       "e1c2": dict(c0=64, c1=0, cout=64, h=H // 2, w=W // 2, pool=True),
       "d0up": dict(c0=64, c1=0, cout=32, h=H // 2, w=W // 2, transposed=True)}[name]
print(name, "%.1f us" % layer(reps=3, **cfg))
