#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs only in the build container (needs /root/reference). It copies
/root/reference/pkg to a scratch dir, builds its Cython backend with the
reference's own setup.py, imports it as ``lidarsplat_ref`` plus the
reference's test oracles (pkg/tests/reference.py, pkg/tests/conftest.py), and
records inputs + outputs as small .npz files. The GPU box never runs this; the
fixtures travel with the repo.

Cases (reference anchors):
  kernels.npz   per-kernel known answers of the native backend
                (_native.pyx:19-297; cf. pkg/tests/test_kernels_parity.py:28-118)
  project.npz   ref_project pure-Python rasterizer (pkg/tests/reference.py:14-72)
                on the 5 scenes of test_projection.py:72-83, plus project_points
  filter.npz    ref_depth_filter_mask (reference.py:175-198) on the 12 configs of
                test_filtering.py:241-254, plus filter_depth_image
  cull.npz      cull_cells (grid.py:131-151) on random grids/views
  pipeline.npz  project_points + depth_filter, culled path (test_kernels_parity.py:121-139)
                and the two-plane scene (conftest.py:64-82)
  c1.json       sha256 digests of the C1 workload (1M uniform box, seed 404,
                512x512, compare_backends.py:23-33) rendered + filtered
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys

import numpy as np

OUT = os.path.dirname(os.path.abspath(__file__))
SCRATCH = "/tmp/lidarsplat_ref_build"


def setup_reference():
    src = "/root/reference/pkg"
    if not os.path.isdir(src):
        sys.exit("needs /root/reference (build container only)")
    if not os.path.isdir(os.path.join(SCRATCH, "src", "lidarsplat_ref")):
        shutil.rmtree(SCRATCH, ignore_errors=True)
        shutil.copytree(src, SCRATCH)
        subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=SCRATCH,
                       check=True, stdout=subprocess.DEVNULL)
        os.rename(os.path.join(SCRATCH, "src", "lidarsplat"),
                  os.path.join(SCRATCH, "src", "lidarsplat_ref"))
    sys.path.insert(0, os.path.join(SCRATCH, "src"))
    # the reference's test helpers import `lidarsplat`; alias it
    import lidarsplat_ref

    sys.modules["lidarsplat"] = lidarsplat_ref
    sys.path.insert(0, os.path.join(SCRATCH, "tests"))
    import conftest as ref_conftest  # noqa: E402
    import reference as ref_oracles  # noqa: E402

    assert "native" in lidarsplat_ref.available_backends()
    return lidarsplat_ref, ref_conftest, ref_oracles


def cam_arrays(cam, prefix, d):
    d[prefix + "rot"] = np.asarray(cam.world_to_camera.rotation, np.float64)
    d[prefix + "t"] = np.asarray(cam.world_to_camera.translation, np.float64)
    d[prefix + "intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.z_near, cam.z_far],
                                  np.float64)
    d[prefix + "wh"] = np.array([cam.width, cam.height], np.int64)


def sparse(rng, h, w, fill=0.5):
    img = np.full((h, w), np.inf, np.float32)
    mask = rng.random((h, w)) < fill
    img[mask] = rng.uniform(0.3, 25.0, size=int(mask.sum())).astype(np.float32)
    return img


def sparse_depth(rng, h, w, fill=0.6, lo=0.5, hi=20.0):
    depth = np.zeros((h, w), np.float32)
    mask = rng.random((h, w)) < fill
    depth[mask] = rng.uniform(lo, hi, size=int(mask.sum())).astype(np.float32)
    return depth


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    L, C, R = setup_reference()
    nat = L.get_backend("native")
    rng = np.random.default_rng(20250218)

    # ---------------- kernels.npz --------------------------------------
    k = {}
    cloud = C.random_cloud(rng, 2000, extent=9.7, offset=-3.3)
    origin = cloud.positions.min(axis=0).astype(np.float64)
    dims = np.array([7, 9, 11], np.int64)
    k["assign_pos"], k["assign_origin"], k["assign_dims"] = cloud.positions, origin, dims
    k["assign_cell"] = np.array(1.37)
    k["assign_ids"] = nat.assign_cells(cloud.positions, origin, 1.37, dims)
    ids = rng.integers(0, 50, size=3000).astype(np.int64)
    k["sort_ids"] = ids
    k["sort_offsets"], k["sort_order"] = nat.counting_sort(ids, 50)
    for s in range(3):
        cl = C.random_cloud(rng, 4000, extent=10.0, offset=-5.0)
        cam = C.random_view(rng, cl)
        starts = np.array([0, 1000, 1000, 2345], np.int64)
        ends = np.array([1000, 1000, 2345, cl.count], np.int64)
        n = int((ends - starts).sum())
        minz = np.full(cam.height * cam.width, np.inf)
        pix = np.empty(n, np.int64)
        z = np.empty(n, np.float64)
        rot, t = cam.world_to_camera.rotation, cam.world_to_camera.translation
        nat.project_min_depth(cl.positions, starts, ends, rot, t, float(cam.fx), float(cam.fy),
                              float(cam.cx), float(cam.cy), cam.width, cam.height,
                              cam.z_near, cam.z_far, minz, pix, z)
        acc = np.zeros((cam.height * cam.width, 4), np.uint64)
        nat.project_accumulate(cl.colors, starts, ends, pix, z, 0.01, minz, acc)
        p = f"proj{s}_"
        k[p + "pos"], k[p + "col"], k[p + "starts"], k[p + "ends"] = (
            cl.positions, cl.colors, starts, ends)
        cam_arrays(cam, p, k)
        k[p + "minz"], k[p + "pix"], k[p + "z"], k[p + "accum"] = minz, pix, z, acc
    for j, shape in enumerate([(8, 8), (13, 21), (16, 5), (3, 3), (1, 7), (31, 2)]):
        img = sparse(rng, *shape)
        k[f"pool{j}_in"], k[f"pool{j}_out"] = img, nat.min_pool_2x2(img)
    for j in range(8):
        img = sparse(rng, int(rng.integers(2, 40)), int(rng.integers(2, 40)))
        thr = float(rng.uniform(0.01, 1.0))
        k[f"lap{j}_in"], k[f"lap{j}_thr"] = img, np.array(thr)
        k[f"lap{j}_out"] = nat.laplacian_edges(img, thr)
    for j in range(8):
        fh, fw = int(rng.integers(2, 40)), int(rng.integers(2, 40))
        fine = sparse(rng, fh, fw)
        coarse = sparse(rng, (fh + 1) // 2, (fw + 1) // 2, fill=0.8)
        edges = nat.laplacian_edges(coarse, 0.25)
        fs = float(rng.uniform(0.0, 2.0))
        k[f"keep{j}_coarse"], k[f"keep{j}_edges"], k[f"keep{j}_fine"] = coarse, edges, fine
        k[f"keep{j}_fs"] = np.array(fs)
        k[f"keep{j}_out"] = nat.filter_keep(coarse, edges, fine, fs)
    for j in range(8):
        fh, fw = int(rng.integers(2, 40)), int(rng.integers(2, 40))
        fine = sparse(rng, fh, fw, fill=0.3)
        coarse = sparse(rng, (fh + 1) // 2, (fw + 1) // 2, fill=0.7)
        k[f"fill{j}_coarse"], k[f"fill{j}_fine"] = coarse, fine
        k[f"fill{j}_out"] = nat.bilinear_fill(coarse, fine)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **k)

    # ---------------- project.npz --------------------------------------
    p = {}
    rng = np.random.default_rng(1234)  # the reference suite's rng fixture seed
    for s in range(5):
        cl = C.random_cloud(rng, 3000, extent=6.0, offset=-3.0)
        cam = C.random_view(rng, cl)
        rgb, depth, alpha = R.ref_project(cl.positions, cl.colors, cam, 0.05)
        fr = L.project_points(cl, None, cam, L.RenderParams(zbuffer_epsilon_rel=0.05))
        assert np.array_equal(fr.rgb, rgb) and np.array_equal(fr.depth, depth)
        q = f"s{s}_"
        p[q + "pos"], p[q + "col"] = cl.positions, cl.colors
        cam_arrays(cam, q, p)
        p[q + "rgb"], p[q + "depth"], p[q + "alpha"] = rgb, depth, alpha
    # hand cases: soft average, occlusion, principal pixel (test_projection.py:20-69)
    np.savez_compressed(os.path.join(OUT, "project.npz"), **p)

    # ---------------- filter.npz ---------------------------------------
    f = {}
    rng = np.random.default_rng(777)
    j = 0
    while j < 16:
        h, w = int(rng.integers(8, 41)), int(rng.integers(8, 41))
        levels = int(rng.integers(1, 5))
        if h < 2**levels or w < 2**levels:
            continue
        depth = sparse_depth(rng, h, w, fill=float(rng.uniform(0.2, 0.9)))
        fs, et = float(rng.uniform(0.0, 1.2)), float(rng.uniform(0.05, 0.6))
        params = L.FilterParams(levels_n=levels, filter_strength=fs, edge_threshold=et)
        keep = L.filter_depth_image(depth, params)
        ref = R.ref_depth_filter_mask(depth.tolist(), levels, fs, et)
        assert np.array_equal(keep, ref)
        q = f"c{j}_"
        f[q + "depth"], f[q + "params"], f[q + "keep"] = (
            depth, np.array([levels, fs, et], np.float64), keep)
        j += 1
    np.savez_compressed(os.path.join(OUT, "filter.npz"), **f)

    # ---------------- cull.npz -----------------------------------------
    c = {}
    rng = np.random.default_rng(101)
    for s in range(6):
        n = int(rng.integers(1000, 20001))
        ext = float(rng.uniform(2.0, 25.0))
        cl = C.random_cloud(rng, n, extent=ext, offset=-ext / 2)
        cam = C.random_view(rng, cl)
        cs = float(rng.uniform(0.5, 2.0))
        grid = L.build_grid(cl, cs)
        q = f"s{s}_"
        c[q + "pos"], c[q + "col"], c[q + "cell"] = cl.positions, cl.colors, np.array(cs)
        cam_arrays(cam, q, c)
        c[q + "planes"] = L.extract_frustum(cam).planes
        c[q + "order"], c[q + "offsets"] = grid.point_order, grid.cell_offsets
        c[q + "culled"] = L.cull_cells(grid, L.extract_frustum(cam))
    np.savez_compressed(os.path.join(OUT, "cull.npz"), **c)

    # ---------------- pipeline.npz -------------------------------------
    q = {}
    rng = np.random.default_rng(4242)
    cl = C.random_cloud(rng, 40_000, extent=8.0)
    cam = C.random_view(rng, cl)
    grid = L.build_grid(cl, 1.0)
    fr = L.project_points(cl, grid, cam, L.RenderParams())
    ft = L.depth_filter(fr, L.FilterParams())
    q["a_pos"], q["a_col"] = cl.positions, cl.colors
    cam_arrays(cam, "a_", q)
    q["a_rgb"], q["a_depth"], q["a_alpha"] = fr.rgb, fr.depth, fr.alpha
    q["a_frgb"], q["a_fdepth"], q["a_falpha"] = ft.rgb, ft.depth, ft.alpha
    cam = C.make_camera()
    cl, checker = C.two_plane_cloud(cam)
    fr = L.project_points(cl, None, cam)
    ft = L.depth_filter(fr, L.FilterParams(levels_n=3, filter_strength=0.5))
    q["b_pos"], q["b_col"], q["b_checker"] = cl.positions, cl.colors, checker
    cam_arrays(cam, "b_", q)
    q["b_rgb"], q["b_depth"], q["b_alpha"] = fr.rgb, fr.depth, fr.alpha
    q["b_falpha"] = ft.alpha
    np.savez_compressed(os.path.join(OUT, "pipeline.npz"), **q)

    # ---------------- c1.json (1M uniform box, 512x512) ------------------
    rng = np.random.default_rng(404)
    npts = 1_000_000
    pts = np.empty((npts, 3), np.float32)
    pts[:, 0] = rng.uniform(-2, 2, npts)
    pts[:, 1] = rng.uniform(-2, 2, npts)
    pts[:, 2] = rng.uniform(5, 13, npts)
    cols = rng.integers(0, 256, (npts, 3), dtype=np.uint8)
    cl = L.PointCloud(pts, cols)
    cam = L.CameraModel(fx=350.0, fy=350.0, cx=256.0, cy=256.0, width=512, height=512)
    grid = L.build_grid(cl, 1.0)
    fr = L.project_points(cl, grid, cam, L.RenderParams())
    ft = L.depth_filter(fr, L.FilterParams())
    info = {
        "inputs": digest(pts, cols),
        "frame": digest(fr.rgb, fr.depth, fr.alpha),
        "filtered": digest(ft.rgb, ft.depth, ft.alpha),
        "filled": int(fr.alpha.sum()),
        "kept": int(ft.alpha.sum()),
        "grid_order": digest(grid.point_order),
        "culled": digest(L.cull_cells(grid, L.extract_frustum(cam))),
    }
    with open(os.path.join(OUT, "c1.json"), "w") as fh:
        json.dump(info, fh, indent=1)
    print("golden fixtures written:", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
