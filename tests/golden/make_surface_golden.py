"""Golden vectors for the reference's public helper surface, produced by
running the REFERENCE (/root/reference/pkg/src/hybridsplat) in the build
container:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_surface_golden.py

Writes tests/golden/surface.npz with
  * build_frame at tile sizes 8 / 16 / 32 (tile_offsets, tile_ids) and the
    SplatFrame arrays t_cam, alpha, view_dir, cam_dist (raster/project.py:
    254-257, 329-379) for the tiny_sh3 and rotcam_sh2 scenes;
  * evaluate_contribution / ray_splat_intersect (project.py:109-152) on
    (splat, pixel) pairs of the rotcam_sh2 frame plus hand-made degenerate
    flat splats;
  * effective_rank, reparameterize_3d_to_2d, modulated_z / modulated_opacity /
    modulated_opacity_grads (exchange.py:58-129);
  * the reference's own finite_diff_check report (grad/findiff.py:78-133) on
    small scenes: its numeric (central-difference) and analytic gradients.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.path.insert(0, HERE)

import hybridsplat as hs  # noqa: E402  (the reference)
from hybridsplat.grad import finite_diff_check as ref_fd  # noqa: E402
from hybridsplat.raster import (RenderSettings, build_frame, evaluate_contribution,  # noqa: E402
                                ray_splat_intersect, DegenerateIntersection, ProjectedSplat)

from make_golden import rotated_camera_scene, to_ref  # noqa: E402
from paper_2512_02932_b200.synthetic import f32_exact, synthetic_scene  # noqa: E402


def main():
    out = {}
    scenes = {"tiny": synthetic_scene(400, 64, 48, 3, seed=1), "rot": rotated_camera_scene()}
    for tag, (sc, cam) in scenes.items():
        rs, rc = to_ref(sc, cam)
        for k, v in (("center", sc.center), ("log_scale", sc.log_scale), ("rotation", sc.rotation),
                     ("opacity_logit", sc.opacity_logit), ("sh", sc.sh_coeffs), ("type", sc.type_spec)):
            out["%s_in_%s" % (tag, k)] = v
        out["%s_cam_intr" % tag] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far])
        out["%s_cam_size" % tag] = np.array([cam.width, cam.height])
        out["%s_cam_w2c" % tag] = cam.world_to_camera
        for t in (8, 16, 32):
            f = build_frame(rs, rc, RenderSettings(tile_size=t))
            out["%s_t%d_tile_offsets" % (tag, t)] = f.tile_offsets
            out["%s_t%d_tile_ids" % (tag, t)] = f.tile_ids
        f = build_frame(rs, rc, RenderSettings())
        for k in ("idx", "t_cam", "alpha", "view_dir", "cam_dist", "valid", "alpha_eff"):
            out["%s_f_%s" % (tag, k)] = getattr(f, k)

    # evaluate_contribution / ray_splat_intersect on real splats of the rotcam frame
    sc, cam = scenes["rot"]
    rs, rc = to_ref(sc, cam)
    f = build_frame(rs, rc, RenderSettings())
    rng = np.random.default_rng(3)
    rows = []
    for k in rng.choice(f.count, size=min(120, f.count), replace=False):
        s = f.splat(int(k))
        for _ in range(3):
            px = (s.screen_center[0] + rng.normal(0, 3.0), s.screen_center[1] + rng.normal(0, 3.0))
            rows.append((s, px, float(f.alpha[k])))
    # hand-made flat splats whose ray/plane solve is exactly singular at
    # some pixels: rows 0 and 1 parallel in their first two columns
    for j in range(6):
        m = np.zeros((3, 4))
        a = rng.normal(size=4)
        m[0] = a
        m[1] = a * (1.0 + j)
        m[1, 3] += 1.0
        m[2] = [0.0, 0.0, 0.0, 1.0]
        s = ProjectedSplat(gaussian_index=j, type_spec=0, screen_center=np.array([5.0, 5.0]),
                           depth_key=1.0, radius=3.0, conic=None, plane_params=m)
        rows.append((s, (5.5, 4.5), 0.7))
    typ, c2, conic, mrow, op, pix, alpha, u, v, deg = ([] for _ in range(10))
    for s, px, o in rows:
        typ.append(s.type_spec)
        c2.append(s.screen_center)
        conic.append([s.conic[0, 0], s.conic[0, 1], s.conic[1, 1]] if s.type_spec == 1 else [0, 0, 0])
        mrow.append(s.plane_params if s.type_spec == 0 else np.zeros((3, 4)))
        op.append(o)
        pix.append(px)
        alpha.append(evaluate_contribution(s, px, o))
        if s.type_spec == 0:
            try:
                uu, vv = ray_splat_intersect(s, px)
                u.append(uu); v.append(vv); deg.append(False)
            except DegenerateIntersection:
                u.append(np.nan); v.append(np.nan); deg.append(True)
        else:
            u.append(np.nan); v.append(np.nan); deg.append(False)
    out.update(ev_typ=np.array(typ, np.uint8), ev_center2d=np.array(c2), ev_conic=np.array(conic),
               ev_mrow=np.array(mrow), ev_opacity=np.array(op), ev_pixel=np.array(pix),
               ev_alpha=np.array(alpha), ev_u=np.array(u), ev_v=np.array(v), ev_degenerate=np.array(deg))

    # exchange helpers
    ls = rng.normal(0.0, 1.0, (300, 3)) * rng.uniform(0.05, 1.5, (300, 1)) - 2.0
    ls[:10] = np.log([[0.5, 0.5, 2.0]] * 10)   # ties
    ls[10:20] = np.log([[2.0, 0.5, 0.5]] * 10)
    rot = rng.normal(size=(300, 4))
    rot /= np.linalg.norm(rot, axis=1, keepdims=True)
    out["ex_log_scale"] = ls
    out["ex_rotation"] = rot
    out["ex_erank"] = hs.exchange.effective_rank(ls)
    rls, rrot = [], []
    for i in range(300):
        g = hs.core.Gaussian(np.zeros(3), ls[i], rot[i], 0.0, np.zeros((3, 1)), 1)
        r = hs.exchange.reparameterize_3d_to_2d(g)
        rls.append(r.log_scale)
        rrot.append(r.rotation)
    out["ex_reparam_log_scale"] = np.array(rls)
    out["ex_reparam_rotation"] = np.array(rrot)
    cfg = hs.exchange.ExchangeConfig()
    lz = np.log(np.concatenate([rng.uniform(0.5, 1.5, 200), [cfg.theta_z, 1.0499, 1.0501, 2.1]]))
    opa = rng.uniform(0.05, 0.99, lz.size)
    out["mod_log_scale_z"] = lz
    out["mod_opacity"] = opa
    out["mod_sz_star"] = hs.exchange.modulated_z(lz, cfg)
    out["mod_alpha_eff"] = hs.exchange.modulated_opacity(opa, lz, cfg)
    da, dl = hs.exchange.modulated_opacity_grads(opa, lz, cfg)
    out["mod_d_alpha"] = da
    out["mod_d_logz"] = dl

    # the reference's own finite-difference oracle on small scenes
    for j, seed in enumerate((5, 6, 7)):
        sc, cam = synthetic_scene(4, 16, 16, 1, seed=seed)
        rs, rc = to_ref(sc, cam)
        target = f32_exact(np.random.default_rng(seed).uniform(0, 1, (16, 16, 3)))
        rep = ref_fd(rs, rc, lambda im: 0.5 * float(np.sum((im - target) ** 2)),
                     lambda im: im - target, 1e-4)
        p = "fd%d_" % j
        for k, v in (("center", sc.center), ("log_scale", sc.log_scale), ("rotation", sc.rotation),
                     ("opacity_logit", sc.opacity_logit), ("sh", sc.sh_coeffs), ("type", sc.type_spec)):
            out[p + "in_" + k] = v
        out[p + "cam_intr"] = np.array([cam.fx, cam.fy, cam.cx, cam.cy, cam.near, cam.far])
        out[p + "cam_w2c"] = cam.world_to_camera
        out[p + "target"] = target
        out[p + "rel_err"] = rep.rel_err
        out[p + "excluded"] = rep.excluded
        out[p + "numeric"] = rep.numeric
        out[p + "analytic"] = rep.analytic
        print("fd scene %d: max rel %.2e, excluded %d" % (j, rep.max_rel_err, int(rep.excluded.sum())))
    path = os.path.join(HERE, "surface.npz")
    np.savez_compressed(path, **out)
    print("surface.npz: %d arrays, %.0f kB" % (len(out), os.path.getsize(path) / 1024))


if __name__ == "__main__":
    main()
