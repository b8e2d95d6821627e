"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package ``hybridsplat`` from
/root/reference/pkg/src, renders / back-propagates / exchanges a set of seeded
scenes, and writes compressed ``.npz`` fixtures next to this script.  The
fixtures pin the CPU oracle (tests/test_oracle_golden.py) and, on the GPU box
where the reference is absent, the CUDA path (tests/test_gpu_*.py).

Scene inputs are float32-representable (synthetic_scene rounds them), so they
are stored as float32 without loss; reference outputs are stored as float64.
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import hybridsplat as hs  # noqa: E402  (the reference)
from hybridsplat.grad import backward as ref_backward  # noqa: E402
from hybridsplat.raster import RenderSettings, render as ref_render  # noqa: E402
from hybridsplat.raster import render_naive as ref_render_naive  # noqa: E402

from paper_2512_02932_b200.synthetic import f32_exact, synthetic_scene  # noqa: E402


def to_ref(scene, cam):
    rs = hs.core.GaussianSet(scene.center, scene.log_scale, scene.rotation,
                             scene.opacity_logit, scene.sh_coeffs, scene.type_spec)
    rc = hs.core.CameraView(cam.fx, cam.fy, cam.cx, cam.cy, cam.width, cam.height,
                            cam.world_to_camera, near=cam.near, far=cam.far)
    return rs, rc


def scene_arrays(scene, cam, st, dt=np.float32):
    """dt = float32 for float32-representable scenes (lossless), float64 for
    the raw-float64 fixtures."""
    return dict(
        in_center=scene.center.astype(dt), in_log_scale=scene.log_scale.astype(dt),
        in_rotation=scene.rotation.astype(dt),
        in_opacity_logit=scene.opacity_logit.astype(dt),
        in_sh=scene.sh_coeffs.astype(dt), in_type=scene.type_spec,
        cam_intr=np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far]),
        cam_size=np.array([cam.width, cam.height]), cam_w2c=cam.world_to_camera,
        background=np.array(st.background, np.float64),
        modulation=np.array([st.theta_z, st.t_z, st.lambda_z]))


def render_fixture(name, scene, cam, st, kg=1, with_log=True, naive=False, seed=11,
                   in_dtype=np.float32):
    rs, rc = to_ref(scene, cam)
    t0 = time.time()
    out = ref_render(rs, rc, st)
    t_fwd = time.time() - t0
    f = out.frame
    data = scene_arrays(scene, cam, st, in_dtype)
    data.update(
        f_idx=f.idx, f_typ=f.typ, f_depth=f.depth, f_center2d=f.center2d, f_cov2d=f.cov2d,
        f_conic=f.conic, f_mrow=f.mrow, f_alpha=f.alpha, f_alpha_eff=f.alpha_eff,
        f_color=f.color, f_bbox=f.bbox, f_radius=f.radius, f_tile_offsets=f.tile_offsets,
        f_tile_ids=f.tile_ids, color=out.color, depth=out.depth,
        transmittance=out.transmittance)
    if with_log:
        lg = out.blend_log
        data.update(log_offsets=lg.offsets, log_pos=lg.position, log_alpha=lg.alpha,
                    log_u=lg.u, log_v=lg.v)
    else:
        data.update(log_counts=np.diff(out.blend_log.offsets).astype(np.int32))
    if naive:
        nv = ref_render_naive(rs, rc, st)
        data.update(naive_color=nv.color, naive_depth=nv.depth,
                    naive_transmittance=nv.transmittance)
    rng = np.random.default_rng(seed)
    pg = f32_exact(rng.normal(size=(kg, cam.height, cam.width, 3)))
    t0 = time.time()
    grads, touched = ref_backward(rs, rc, out, pg)
    t_bwd = time.time() - t0
    data.update(pixel_grad=pg.astype(np.float32),
                grads=np.stack([g.flat() for g in grads]), touched=touched)
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **data)
    print("%-14s N=%-6d M=%-6d K=%-7d fwd %.1fs bwd %.1fs -> %s (%.0f kB)"
          % (name, scene.count, f.count, f.tile_ids.size, t_fwd, t_bwd, os.path.basename(path),
             os.path.getsize(path) / 1024))


def stress2d_scene(seed=5, n=60, size=48):
    """Large, tilted, near-camera 2D surfels: exercises the dual-conic AABB and
    its full-screen fallback ('Hard parts')."""
    from paper_2512_02932_b200.core import GaussianSet
    from paper_2512_02932_b200.synthetic import synthetic_camera
    rng = np.random.default_rng(seed)
    cam = synthetic_camera(size, size)
    z = rng.uniform(0.3, 3.0, n)
    px = rng.uniform(-0.2 * size, 1.2 * size, n)
    py = rng.uniform(-0.2 * size, 1.2 * size, n)
    center = np.stack([(px - cam.cx) * z / cam.fx, (py - cam.cy) * z / cam.fy, z], 1)
    ls = np.log(rng.uniform(0.05, 0.8, (n, 3)))
    rot = rng.normal(size=(n, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    sc = GaussianSet(f32_exact(center), f32_exact(ls), f32_exact(rot),
                     f32_exact(rng.normal(size=n)), f32_exact(rng.normal(0, .3, (n, 3, 4))),
                     np.zeros(n, np.uint8))
    return sc, cam


def rotated_camera_scene(seed=7):
    """Non-identity world-to-camera: exercises V in projection and chain rule."""
    from paper_2512_02932_b200.synthetic import synthetic_camera
    sc, cam = synthetic_scene(500, 64, 48, 2, seed=seed)
    ang = 0.3
    Rz = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1]])
    Rx = np.array([[1, 0, 0], [0, np.cos(0.2), -np.sin(0.2)], [0, np.sin(0.2), np.cos(0.2)]])
    R = Rx @ Rz
    w2c = np.eye(4)
    w2c[:3, :3] = R
    w2c[:3, 3] = [0.05, -0.1, 0.2]
    # Move the scene so it stays in view: x_world = R^T (x_cam - t)
    xc = sc.center
    sc.center[:] = f32_exact((xc - w2c[:3, 3]) @ R)
    return sc, synthetic_camera(64, 48, w2c)


def _mat_to_quat(R):
    """Rotation matrix -> w-first unit quaternion (Shepperd, w >= 0)."""
    q = np.empty(4)
    tr = np.trace(R)
    if tr > 0:
        t = np.sqrt(tr + 1.0) * 2
        q[:] = [0.25 * t, (R[2, 1] - R[1, 2]) / t, (R[0, 2] - R[2, 0]) / t, (R[1, 0] - R[0, 1]) / t]
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        t = np.sqrt(1.0 + R[i, i] - R[j, j] - R[k, k]) * 2
        q[0] = (R[k, j] - R[j, k]) / t
        q[1 + i] = 0.25 * t
        q[1 + j] = (R[j, i] + R[i, j]) / t
        q[1 + k] = (R[k, i] + R[i, k]) / t
    return q if q[0] >= 0 else -q


def grazing_scene(seed=23, n=160, size=64):
    """2D surfels seen almost edge-on: each surfel's first tangent axis is the
    view ray through its centre, tilted by 1e-4 .. 0.3 rad, so the ray/plane
    2x2 solve is near-degenerate (|den| close to its float32 error bound) over
    much of its footprint.  Mixed with a few 3D Gaussians behind them."""
    from paper_2512_02932_b200.core import GaussianSet
    from paper_2512_02932_b200.synthetic import synthetic_camera
    rng = np.random.default_rng(seed)
    cam = synthetic_camera(size, size)
    z = rng.uniform(0.8, 4.0, n)
    px = rng.uniform(0.1 * size, 0.9 * size, n)
    py = rng.uniform(0.1 * size, 0.9 * size, n)
    center = np.stack([(px - cam.cx) * z / cam.fx, (py - cam.cy) * z / cam.fy, z], 1)
    rot = np.zeros((n, 4))
    ty = np.zeros(n, np.uint8)
    ty[n - n // 5:] = 1
    for i in range(n):
        if i % 2 == 0:
            d = center[i] / np.linalg.norm(center[i])
        else:
            # the plane contains the ray through a pixel centre near the
            # splat: that pixel's ray/plane solve is exactly singular
            qx = np.floor(px[i]) + rng.integers(-3, 4) + 0.5
            qy = np.floor(py[i]) + rng.integers(-3, 4) + 0.5
            d = np.array([(qx - cam.cx) / cam.fx, (qy - cam.cy) / cam.fy, 1.0])
            d /= np.linalg.norm(d)
        a = rng.normal(size=3)
        a -= d * (a @ d)
        a /= np.linalg.norm(a)
        ang = 10.0 ** rng.uniform(-4, np.log10(0.3)) if i % 2 == 0 else 0.0
        t0 = np.cos(ang) * d + np.sin(ang) * np.cross(a, d)   # ~ the view ray
        t1 = a
        nrm = np.cross(t0, t1)
        R = np.stack([t0, t1, nrm], 1)
        if rng.random() < 0.5:
            R = R[:, [1, 0, 2]] * np.array([1, 1, -1])           # swap tangents (det +1)
        rot[i] = _mat_to_quat(R)
    ls = np.log(np.stack([rng.uniform(0.05, 0.4, n), rng.uniform(0.05, 0.4, n),
                          rng.uniform(0.01, 0.05, n)], 1))
    sc = GaussianSet(f32_exact(center), f32_exact(ls), f32_exact(rot),
                     f32_exact(rng.normal(1.0, 1.0, n)), f32_exact(rng.normal(0, .3, (n, 3, 4))), ty)
    return sc, cam


def raw_f64_scene(seed=17):
    """A scene whose float64 inputs are NOT float32-representable, with a
    rotated, translated camera (so view depths are not exact either): the
    float32 rounding of these inputs gives a different depth order and
    different tile lists, so only a float64-faithful path matches the
    reference's frame arrays bit for bit."""
    sc, _ = synthetic_scene(3000, 128, 96, 1, seed=seed, f32=False)
    ang = 0.2
    R = np.array([[np.cos(ang), -np.sin(ang), 0], [np.sin(ang), np.cos(ang), 0], [0, 0, 1]])
    w2c = np.eye(4)
    w2c[:3, :3] = R
    w2c[:3, 3] = [0.013, -0.027, 0.11]
    sc.center[:] = (sc.center - w2c[:3, 3]) @ R
    # near-ties in depth below float32 resolution: pairs of Gaussians whose
    # view depths differ by ~1e-9 (float32 rounding merges or swaps them)
    k = 200
    sc.center[1:2 * k:2] = sc.center[0:2 * k:2] + 1e-9 * np.random.default_rng(seed).normal(size=(k, 3))
    from paper_2512_02932_b200.synthetic import synthetic_camera
    return sc, synthetic_camera(128, 96, w2c)


def exchange_f64_fixture():
    """exchange_pass on raw float64 scales (not float32-representable), with
    rows placed within 1e-12 of the erank threshold."""
    rng = np.random.default_rng(19)
    n = 3000
    ls = rng.normal(0.0, 1.0, (n, 3)) * rng.uniform(0.05, 1.5, (n, 1)) - 2.0
    ls[:40] = np.log([[1.0, 1.0, 2.6]] * 40) + rng.normal(0, 0.003, (40, 3))
    rot = rng.normal(size=(n, 4))
    rot = rot / np.linalg.norm(rot, axis=1, keepdims=True)
    ty = (rng.random(n) < 0.5).astype(np.uint8)
    sc = hs.core.GaussianSet(np.zeros((n, 3)), ls.copy(), rot.copy(), np.zeros(n),
                             np.zeros((n, 3, 1)), ty.copy())
    rep = hs.exchange.exchange_pass(sc, hs.exchange.ExchangeConfig())
    np.savez_compressed(os.path.join(HERE, "exchange_f64.npz"),
                        in_log_scale=ls, in_rotation=rot, in_type=ty, out_log_scale=sc.log_scale,
                        out_rotation=sc.rotation, out_type=sc.type_spec,
                        eranks=hs.exchange.effective_rank(ls),
                        counts=np.array([rep.n_3d_to_2d, rep.n_2d_to_3d, rep.n_2d, rep.n_3d]),
                        hist=rep.erank_hist, edges=rep.erank_edges)
    print("exchange_f64: demoted %d promoted %d" % (rep.n_3d_to_2d, rep.n_2d_to_3d))


def exchange_fixture():
    rng = np.random.default_rng(13)
    n = 4000
    ls = f32_exact(rng.normal(0.0, 1.0, (n, 3)) * rng.uniform(0.05, 1.5, (n, 1)) - 2.0)
    # a block of near-threshold rows and exact ties for choose_permutation
    ls[:50] = f32_exact(np.log([[1.0, 1.0, 2.6]] * 50) + rng.normal(0, 0.01, (50, 3)))
    ls[50:60] = f32_exact(np.log(np.array([[0.5, 0.5, 2.0]] * 10)))
    ls[60:70] = f32_exact(np.log(np.array([[2.0, 0.5, 0.5]] * 10)))
    rot = rng.normal(size=(n, 4))
    rot = f32_exact(rot / np.linalg.norm(rot, axis=1, keepdims=True))
    ty = (rng.random(n) < 0.5).astype(np.uint8)
    sc = hs.core.GaussianSet(np.zeros((n, 3)), ls.copy(), rot.copy(), np.zeros(n),
                             np.zeros((n, 3, 1)), ty.copy())  # the reference aliases f64 inputs
    rep = hs.exchange.exchange_pass(sc, hs.exchange.ExchangeConfig())
    np.savez_compressed(os.path.join(HERE, "exchange.npz"),
                        in_log_scale=ls.astype(np.float32), in_rotation=rot.astype(np.float32),
                        in_type=ty, out_log_scale=sc.log_scale, out_rotation=sc.rotation,
                        out_type=sc.type_spec, eranks=hs.exchange.effective_rank(ls),
                        counts=np.array([rep.n_3d_to_2d, rep.n_2d_to_3d, rep.n_2d, rep.n_3d]),
                        hist=rep.erank_hist, edges=rep.erank_edges)
    print("exchange: demoted %d promoted %d" % (rep.n_3d_to_2d, rep.n_2d_to_3d))


def main(which=None):
    jobs = {
        "tiny_sh3": lambda: render_fixture(
            "tiny_sh3", *synthetic_scene(400, 64, 48, 3, seed=1),
            RenderSettings(background=(0.1, 0.2, 0.3)), kg=2, naive=True),
        "stress2d": lambda: render_fixture(
            "stress2d", *stress2d_scene(), RenderSettings(background=(0.0, 0.5, 1.0)), kg=1,
            naive=True),
        "rotcam_sh2": lambda: render_fixture(
            "rotcam_sh2", *rotated_camera_scene(), RenderSettings(), kg=3),
        "c1": lambda: render_fixture(
            "c1", *synthetic_scene(10_000, 256, 256, 0, seed=0), RenderSettings(), kg=1,
            with_log=False),
        "exchange": exchange_fixture,
        "raw_f64": lambda: render_fixture(
            "raw_f64", *raw_f64_scene(), RenderSettings(background=(0.3, 0.1, 0.2)), kg=1, with_log=False,
            in_dtype=np.float64),
        "exchange_f64": exchange_f64_fixture,
        "grazing": lambda: render_fixture(
            "grazing", *grazing_scene(), RenderSettings(background=(0.2, 0.2, 0.2)), kg=1,
            naive=True),
    }
    for name, fn in jobs.items():
        if which and name not in which:
            continue
        fn()


if __name__ == "__main__":
    main(sys.argv[1:])
