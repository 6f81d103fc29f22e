#!/usr/bin/env python3
"""PLY loader fixtures FROM THE REFERENCE ITSELF (build container only).

Builds a set of PLY byte strings (ascii / binary, extra properties, elements
before and after the vertex block, and malformed variants) and records what
the reference's pure-Python ``lidarsplat.io.ply.load_ply`` returns for each:
the cloud's arrays, or the PlyParseError message + byte offset
(R:io/ply.py:154-199).  Also records the reference's save_ply bytes.

    python tests/golden/make_ply_golden.py  ->  tests/golden/ply.npz
"""

import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from lidarsplat.cloud import PointCloud  # noqa: E402  (the reference's)
from lidarsplat.errors import PlyParseError  # noqa: E402
from lidarsplat.io.ply import load_ply, save_ply  # noqa: E402

rng = np.random.default_rng(5)
n = 37
pos = (rng.random((n, 3)) * 40 - 20).astype(np.float32)
col = rng.integers(0, 256, (n, 3), dtype=np.uint8)
cloud = PointCloud(pos, col)


def header(fmt, body):
    return (f"ply\nformat {fmt} 1.0\ncomment made by make_ply_golden\n{body}end_header\n").encode()


VERT = ("element vertex {n}\nproperty float x\nproperty float y\nproperty float z\n"
        "property uchar red\nproperty uchar green\nproperty uchar blue\n")
cases = {}
with tempfile.TemporaryDirectory() as d:
    for b in (True, False):
        p = os.path.join(d, "c.ply")
        save_ply(cloud, p, binary=b)
        cases[f"saved_{'bin' if b else 'ascii'}"] = open(p, "rb").read()
# extra properties, interleaved order, a preceding fixed-size element, a trailing element
rec = np.empty(n, dtype=[("nx", "<f4"), ("x", "<f4"), ("y", "<f4"), ("z", "<f4"),
                         ("intensity", "<u2"), ("red", "u1"), ("green", "u1"), ("blue", "u1"),
                         ("t", "<f8")])
for i, a in enumerate("xyz"):
    rec[a] = pos[:, i]
for i, a in enumerate(("red", "green", "blue")):
    rec[a] = col[:, i]
rec["nx"] = 1.0
rec["intensity"] = 7
rec["t"] = 0.5
pre = np.array([(1, 2.0), (3, 4.0)], dtype=[("a", "<i4"), ("b", "<f4")])
body = ("element meta 2\nproperty int a\nproperty float b\n"
        f"element vertex {n}\nproperty float nx\nproperty float x\nproperty float y\n"
        "property float z\nproperty ushort intensity\nproperty uchar red\n"
        "property uchar green\nproperty uchar blue\nproperty double t\n"
        "element face 1\nproperty list uchar int vertex_indices\n")
cases["bin_extras"] = header("binary_little_endian", body) + pre.tobytes() + rec.tobytes() + b"\x03\x00"
lines = "".join(f"{float(r['nx'])} {float(r['x'])!r} {float(r['y'])!r} {float(r['z'])!r} "
                f"{int(r['intensity'])} {int(r['red'])} {int(r['green'])} {int(r['blue'])} "
                f"{float(r['t'])}\n" for r in rec)
cases["ascii_extras"] = (header("ascii", body) + b"1 2.0\n3 4.0\n" + lines.encode() + b"3 0 1 2\n")
v = VERT.format(n=n)
cases["bin_truncated"] = header("binary_little_endian", v) + rec[["x", "y", "z"]].tobytes()[:50]
good_ascii = header("ascii", v) + "".join(f"{p[0]} {p[1]} {p[2]} {c[0]} {c[1]} {c[2]}\n"
                                          for p, c in zip(pos, col)).encode()
cases["ascii_bad_color"] = good_ascii.replace(f" {col[5][1]} {col[5][2]}\n".encode(),
                                              f" 300 {col[5][2]}\n".encode(), 1)
cases["ascii_short_line"] = good_ascii.rsplit(b"\n", 3)[0] + b"\n1 2\n"
cases["ascii_truncated"] = good_ascii.rsplit(b"\n", 4)[0] + b"\n"
hdr_end = good_ascii.index(b"end_header\n") + len(b"end_header\n")
body_lines = good_ascii[hdr_end:].split(b"\n")
body_lines[3] = b"foo bar baz 1 2 3"
cases["ascii_garbage"] = good_ascii[:hdr_end] + b"\n".join(body_lines)
cases["no_magic"] = b"plx\n" + good_ascii[4:]
cases["big_endian"] = header("binary_big_endian", v)
cases["bad_format"] = b"ply\nformat ascii 2.0\nend_header\n"
cases["no_format"] = b"ply\n" + v.encode() + b"end_header\n"
cases["no_vertex"] = header("ascii", "element meta 1\nproperty int a\n")
cases["empty"] = header("ascii", VERT.format(n=0))
cases["double_x"] = header("ascii", v.replace("float x", "double x"))
cases["missing_blue"] = header("ascii", v.replace("property uchar blue\n", ""))
cases["list_vertex"] = header("ascii", v + "property list uchar int idx\n")
cases["unknown_type"] = header("ascii", v.replace("uchar red", "ufoo red"))
cases["bad_line"] = header("ascii", v + "wibble\n")
cases["prop_first"] = b"ply\nformat ascii 1.0\nproperty float x\nend_header\n"
cases["no_end"] = header("ascii", v)[:-len("end_header\n")]
cases["list_before_vertex"] = header("binary_little_endian",
                                     "element face 1\nproperty list uchar int i\n" + v)

out = {}
with tempfile.TemporaryDirectory() as d:
    for name, data in cases.items():
        p = os.path.join(d, name + ".ply")
        with open(p, "wb") as f:
            f.write(data)
        out[f"{name}__bytes"] = np.frombuffer(data, np.uint8)
        try:
            c = load_ply(p)
            out[f"{name}__pos"], out[f"{name}__col"] = c.positions, c.colors
        except PlyParseError as e:
            out[f"{name}__err"] = np.array(str(e))
            out[f"{name}__off"] = np.array(e.offset)
        except Exception as e:  # noqa: BLE001
            out[f"{name}__other"] = np.array(type(e).__name__)
np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ply.npz"), **out)
for name in cases:
    tag = "ok" if f"{name}__pos" in out else (str(out.get(f"{name}__err", out.get(f"{name}__other"))))
    print(f"{name:20s} {tag}")
