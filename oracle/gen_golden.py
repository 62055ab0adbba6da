"""Generate tests/golden/*.npz by running the REFERENCE itself -- test infrastructure.

Run in the build container only (it imports ``voldiff`` from
/root/reference/pkg/src, which does not exist on the GPU box):

    python oracle/gen_golden.py

Every fixture stores the reference's fp64 outputs for fp32-representable inputs
so that (a) ``tests/test_oracle_golden.py`` pins ``oracle/dvr_oracle.py`` to the
reference on CPU, and (b) the ``-m gpu`` parity tests compare the CUDA path to
the same numbers.  Large gradients (C4/C5 row bands) are stored sparsely.

Cases (reference call sites in brackets):
* kat_*      known-answer scenes of test_renderer.py:98-122, 166-175, 251-259
* rand_*     gradcheck.random_scene (gradcheck.py:44-68) with L1 seeds, all four
             targets, inversion and stored memory modes (renderer.py:491-685)
* C1         the full C1 view: image + every target, dense N(0,1) seed
* C2..C5     row bands of view 0: image band, n_steps, and the config's targets
* counts     exact per-config sample totals (renderer.py:209-214)
* C4_step_*, C5_step_*  the fused tomography step at config scale (row bands of a
             few views): reference images, band images, L1 loss, density gradient
* C1_step_*, C2_step_*  the fused TF-target steps (C1 full view, C2 bands): loss, d_tf
             (and C1's d_volume)
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import voldiff as vd                                   # noqa: E402  (the reference)
from voldiff import renderer as vr                     # noqa: E402
from voldiff.gradcheck import random_scene             # noqa: E402

from paper_2107_12672_b200.scenes import CONFIGS       # noqa: E402

TARGETS = ("tf", "volume", "camera", "stepsize")
BANDS = {"C2": (120, 136), "C3": (250, 258), "C4": (254, 258), "C5": (510, 512)}


def f32(a):
    return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)


def grads_of(gs, target):
    return {"tf": gs.d_tf, "volume": gs.d_volume, "camera": gs.d_camera,
            "stepsize": np.array([gs.d_stepsize]) if gs.d_stepsize is not None else None}[target]


def cam_fields(cam):
    return np.array([cam.lon_deg, cam.lat_deg, cam.radius, *cam.center, cam.fov_y_deg,
                     cam.width, cam.height], np.float64)


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1024:.0f} KiB)")


def scene_case(name, volume, texels, cam, dt, seed, targets=TARGETS, modes=("inversion",),
               early=True, box=((-0.5, -0.5, -0.5), (0.5, 0.5, 0.5))):
    volume, texels, seed = f32(volume), f32(texels), f32(seed)
    V = vd.DensityVolume(volume, np.array(box[0]), np.array(box[1]))
    T = vd.TransferFunction(texels)
    out = dict(volume=volume.astype(np.float32), texels=texels.astype(np.float32),
               box=np.array(box, np.float64), cam=cam_fields(cam), dt=np.float64(dt),
               seed=seed)
    if early:
        out["image_none"] = vd.render(V, T, cam, vd.RenderConfig(dt=dt)).data
    img = vd.render(V, T, cam, vd.RenderConfig(dt=dt, target="volume")).data
    out["image"] = img
    u, v = vr._tile_pixels(cam, 0, cam.height)
    _, _, slab = vr._ray_setup(("density", V, T), cam, u, v)
    out["n_steps"] = vr._step_counts(slab[0], slab[1], dt, slab[4]).astype(np.int32)
    for mode in modes:
        for t in targets:
            gs = vd.render_adjoint(V, T, cam, vd.RenderConfig(dt=dt, target=t, memory_mode=mode),
                                   seed)
            out[f"{mode}_{t}"] = np.asarray(grads_of(gs, t), np.float64)
            out[f"{mode}_{t}_state_floats"] = np.int64(gs.state_floats)
    save(name, **out)


def kat_cases():
    ones = np.ones((8, 8, 8))
    cam = vd.SphericalCamera(0.0, 0.0, 2.0, fov_y_deg=8.0, width=9, height=9)
    seed = np.ones((9, 9, 4))
    for tau0 in (0.1, 1.0, 10.0):               # test_renderer.py:105-112
        scene_case(f"kat_transparency_{tau0:g}", ones, np.tile([0.5, 0.5, 0.5, tau0], (2, 1)),
                   cam, 0.05, seed)
    scene_case("kat_emission", ones, np.tile([0.7, 0.7, 0.7, 2.0], (2, 1)), cam, 0.01, seed)
    scene_case("kat_stepsize", ones, np.tile([0.4, 0.4, 0.4, 1.3], (2, 1)), cam, 0.05, seed)
    scene_case("kat_empty", np.zeros((4, 4, 4)), np.array([[0, 0, 0, 0], [1, 1, 1, 2.0]]),
               vd.SphericalCamera(10.0, 5.0, 2.0, width=6, height=6), 0.05, np.ones((6, 6, 4)))
    scene_case("kat_miss", np.ones((4, 4, 4)), np.tile([1.0, 1.0, 1.0, 5.0], (2, 1)),
               vd.SphericalCamera(0.0, 80.0, 50.0, fov_y_deg=0.5, width=4, height=4), 0.1,
               np.ones((4, 4, 4)))
    rng = np.random.default_rng(42)             # conftest.py:20-41 fixtures
    small_tf = np.column_stack([rng.uniform(0.05, 1.0, (8, 3)), rng.uniform(0.3, 2.0, 8)])
    scene_case("kat_untouched", np.full((8, 8, 8), 0.5), f32(small_tf),
               vd.SphericalCamera(0.0, 0.0, 2.0, fov_y_deg=2.0, width=4, height=4), 0.05,
               np.ones((4, 4, 4)), targets=("volume",))
    # non-cubic grid, off-centre box, non-square image, camera off-centre
    rng = np.random.default_rng(7)
    vol = f32(rng.uniform(0.05, 0.95, (6, 9, 5)))
    tex = f32(np.column_stack([rng.uniform(0.05, 1, (5, 3)), rng.uniform(0.3, 2.5, 5)]))
    cam = vd.SphericalCamera(200.0, -35.0, 2.2, center=np.array([0.1, -0.05, 0.2]),
                             fov_y_deg=40.0, width=11, height=7)
    scene_case("kat_anisotropic", vol, tex, cam, 0.037,
               f32(rng.normal(size=(7, 11, 4))), modes=("inversion", "stored"),
               box=((-0.4, -0.6, -0.3), (0.6, 0.5, 0.7)))
    # R = 1 and R = 2 transfer functions
    for R in (1, 2):
        tex = f32(np.column_stack([rng.uniform(0.05, 1, (R, 3)), rng.uniform(0.3, 2.5, R)]))
        scene_case(f"kat_tf_r{R}", f32(rng.uniform(0.1, 0.9, (8, 8, 8))), tex,
                   vd.SphericalCamera(40.0, 10.0, 2.5, width=8, height=8), 0.06,
                   f32(rng.normal(size=(8, 8, 4))))


def random_cases():
    for s, R in ((500, 8), (501, 8), (502, 2), (503, 8), (2000, 2), (2001, 8)):
        sc = random_scene(s, tf_res=R)
        vol, tex = f32(sc.volume.values), f32(sc.tf.texels)
        V, T = vd.DensityVolume(vol), vd.TransferFunction(tex)
        img = vd.render(V, T, sc.cam, vd.RenderConfig(dt=sc.dt, target="volume"))
        _, seeds = vd.l1_loss([img], [sc.ref])
        scene_case(f"rand_{s}", vol, tex, sc.cam, sc.dt, seeds[0],
                   modes=("inversion", "stored"))


def config_cases():
    rng = np.random.default_rng(1234)
    for name in ("C1", "C2", "C3", "C4", "C5"):
        c = CONFIGS[name]
        t0 = time.time()
        vol = c.volume().astype(np.float64)
        tex = f32(c.texels())
        V, T = vd.DensityVolume(vol), vd.TransferFunction(tex)
        lon, lat = c.view_poses()[0]
        cam = vd.SphericalCamera(lon, lat, c.radius, fov_y_deg=c.fov, width=c.image,
                                 height=c.image)
        r0, r1 = BANDS.get(name, (0, c.image))
        scene = ("density", V, T)
        out = dict(texels=tex.astype(np.float32), cam=cam_fields(cam), dt=np.float64(c.dt),
                   rows=np.array([r0, r1]),
                   volume_sum=np.float64(vol.sum()),
                   volume_probe=vol.reshape(-1)[:: max(1, vol.size // 4096)].copy())
        u, v = vr._tile_pixels(cam, r0, r1)
        o, w, slab = vr._ray_setup(scene, cam, u, v)
        n = vr._step_counts(slab[0], slab[1], c.dt, slab[4])
        out["n_steps"] = n.astype(np.int32)
        out["tn_tf"] = np.stack([slab[0], slab[1]]).astype(np.float64)
        band, _ = vr._march_fused(scene, o, w, c.dt, slab, n)
        out["image"] = band.reshape(r1 - r0, c.image, 4)
        seed = np.zeros((c.image, c.image, 4))
        seed[r0:r1] = rng.normal(size=(r1 - r0, c.image, 4))
        out["seed_band"] = seed[r0:r1].copy()
        targets = TARGETS if name == "C1" else c.targets
        for t in targets:
            gs = vr._adjoint_tile(scene, cam, vd.RenderConfig(dt=c.dt, target=t),
                                  seed[r0:r1].reshape(-1, 4), (r0, r1),
                                  final_rgba=band)
            g = np.asarray(grads_of(gs, t), np.float64)
            if t == "volume" and name != "C1":
                nz = np.flatnonzero(g)
                out["inversion_volume_idx"] = nz.astype(np.int64)
                out["inversion_volume_val"] = g.reshape(-1)[nz]
            else:
                out[f"inversion_{t}"] = g
        save(name, **out)
        print(f"  {name}: {time.time() - t0:.1f}s, band samples {int(n.sum())}")


# fused-step fixtures at config scale: (views, rows) of each case
STEP_BANDS = {"C4": ((0, 17), (252, 260)), "C5": ((0,), (508, 516))}


def step_cases():
    """The tomography step the bench times (tasks.py:397-432: render -> l1_loss ->
    render_adjoint), at the config's full volume and image size on row bands of a few
    views, computed by the reference: reference images rendered from the truth, the
    estimate's band images, the L1 loss over the bands (objectives.py:38-54, count =
    the bands' element count) and the density gradient of that loss.  Estimates:
    ``dense`` = 0.85 truth + 0.1 U(0,1) (iteration 1 of the bench, no exact zeros) and,
    for C4, ``sparse`` = the truth's support only (exact zeros outside the object,
    what the optimisation grows, so the band tape's empty-space skips run)."""
    rng = np.random.default_rng(99)
    for name, (views, (r0, r1)) in STEP_BANDS.items():
        c = CONFIGS[name]
        truth = c.volume().astype(np.float64)
        tex = f32(c.texels())
        ests = {"dense": f32(0.85 * truth + 0.1 * rng.uniform(size=truth.shape))}
        if name == "C4":
            ests["sparse"] = f32(np.where(truth > 0, np.clip(0.7 * truth + 0.05, 0, 1), 0.0))
        T = vd.TransferFunction(tex)
        poses = c.view_poses()
        cams = [vd.SphericalCamera(*poses[k], c.radius, fov_y_deg=c.fov, width=c.image,
                                   height=c.image) for k in views]
        count = 4 * c.image * (r1 - r0) * len(views)
        refs = []
        for cam in cams:
            u, v = vr._tile_pixels(cam, r0, r1)
            scene = ("density", vd.DensityVolume(truth), T)
            o, w, slab = vr._ray_setup(scene, cam, u, v)
            n = vr._step_counts(slab[0], slab[1], c.dt, slab[4])
            band, _ = vr._march_fused(scene, o, w, c.dt, slab, n)
            refs.append(band)
        for kind, est in ests.items():
            t0 = time.time()
            scene = ("density", vd.DensityVolume(est), T)
            imgs, loss, grad = [], 0.0, np.zeros(est.size)
            for cam, ref in zip(cams, refs):
                u, v = vr._tile_pixels(cam, r0, r1)
                o, w, slab = vr._ray_setup(scene, cam, u, v)
                n = vr._step_counts(slab[0], slab[1], c.dt, slab[4])
                band, _ = vr._march_fused(scene, o, w, c.dt, slab, n)
                loss += float(np.abs(band - ref).sum()) / count     # objectives.py:51-53
                seed = np.sign(band - ref) / count
                gs = vr._adjoint_tile(scene, cam, vd.RenderConfig(dt=c.dt, target="volume"),
                                      seed, (r0, r1), final_rgba=band)
                grad += np.asarray(gs.d_volume, np.float64).reshape(-1)
                imgs.append(band.reshape(r1 - r0, c.image, 4))
            nz = np.flatnonzero(grad)
            # the estimate is rebuilt by the test from the same generator: store a probe
            save(f"{name}_step_{kind}", views=np.array(views), rows=np.array([r0, r1]),
                 texels=tex.astype(np.float32), dt=np.float64(c.dt), count=np.float64(count),
                 refs=np.stack(refs).reshape(len(views), r1 - r0, c.image, 4).astype(np.float32),
                 image=np.stack(imgs), loss=np.float64(loss),
                 est_probe=est.reshape(-1)[:: max(1, est.size // 4096)].copy(),
                 volume_idx=nz.astype(np.int32), volume_val=grad[nz].astype(np.float32))
            print(f"  {name} {kind}: {time.time() - t0:.1f}s, loss {loss:.6g}")


# the fused TF-target steps (C1: volume + tf, full view; C2: tf, row bands of two views)
TF_STEP_BANDS = {"C1": ((0,), (0, 128)), "C2": ((0, 5), (120, 136))}


def tf_step_cases():
    """The fused step of the TF-target configs as the bench runs it (ShardedStep:
    forward -> l1_loss -> render_adjoint per view, tasks.py:258-270 / 397-432) at the
    configs' full sizes, computed by the reference: references rendered from the truth,
    the dense estimate 0.85 truth + 0.1 U(0,1) (its own default_rng(77) stream, C1 then
    C2), the L1 loss over the bands and the gradients of the config's targets."""
    rng = np.random.default_rng(77)
    for name, (views, (r0, r1)) in TF_STEP_BANDS.items():
        t0 = time.time()
        c = CONFIGS[name]
        truth = c.volume().astype(np.float64)
        est = f32(0.85 * truth + 0.1 * rng.uniform(size=truth.shape))
        tex = f32(c.texels())
        T = vd.TransferFunction(tex)
        poses = c.view_poses()
        cams = [vd.SphericalCamera(*poses[k], c.radius, fov_y_deg=c.fov, width=c.image,
                                   height=c.image) for k in views]
        count = 4 * c.image * (r1 - r0) * len(views)
        refs, imgs, loss = [], [], 0.0
        grads = {t: None for t in c.targets}
        for cam in cams:
            u, v = vr._tile_pixels(cam, r0, r1)
            scene = ("density", vd.DensityVolume(truth), T)
            o, w, slab = vr._ray_setup(scene, cam, u, v)
            n = vr._step_counts(slab[0], slab[1], c.dt, slab[4])
            ref, _ = vr._march_fused(scene, o, w, c.dt, slab, n)
            scene = ("density", vd.DensityVolume(est), T)
            o, w, slab = vr._ray_setup(scene, cam, u, v)
            band, _ = vr._march_fused(scene, o, w, c.dt, slab, n)
            loss += float(np.abs(band - ref).sum()) / count
            seed = np.sign(band - ref) / count
            for t in c.targets:
                gs = vr._adjoint_tile(scene, cam, vd.RenderConfig(dt=c.dt, target=t), seed,
                                      (r0, r1), final_rgba=band)
                g = np.asarray(grads_of(gs, t), np.float64)
                grads[t] = g if grads[t] is None else grads[t] + g
            refs.append(ref)
            imgs.append(band.reshape(r1 - r0, c.image, 4))
        out = dict(views=np.array(views), rows=np.array([r0, r1]), texels=tex.astype(np.float32),
                   dt=np.float64(c.dt), count=np.float64(count),
                   refs=np.stack(refs).reshape(len(views), r1 - r0, c.image, 4).astype(np.float32),
                   image=np.stack(imgs), loss=np.float64(loss),
                   est_probe=est.reshape(-1)[:: max(1, est.size // 4096)].copy(),
                   d_tf=grads["tf"])
        if "volume" in grads:
            nz = np.flatnonzero(grads["volume"])
            out["volume_idx"] = nz.astype(np.int32)
            out["volume_val"] = grads["volume"].reshape(-1)[nz].astype(np.float32)
        save(f"{name}_step_dense", **out)
        print(f"  {name}: {time.time() - t0:.1f}s, loss {loss:.6g}")


def count_cases():
    out = {}
    for name, c in CONFIGS.items():
        vol = vd.DensityVolume(np.zeros((2, 2, 2)))
        total = 0
        rays = 0
        for lon, lat in c.view_poses():
            cam = vd.SphericalCamera(lon, lat, c.radius, fov_y_deg=c.fov, width=c.image,
                                     height=c.image)
            for r0 in range(0, c.image, 256):
                r1 = min(r0 + 256, c.image)
                u, v = vr._tile_pixels(cam, r0, r1)
                _, _, slab = vr._ray_setup(("density", vol, None), cam, u, v)
                total += int(vr._step_counts(slab[0], slab[1], c.dt, slab[4]).sum())
                rays += u.shape[0]
        out[name + "_samples"] = np.int64(total)
        out[name + "_rays"] = np.int64(rays)
        print(f"  {name}: {rays} rays, {total} samples")
    save("counts", **out)


def color_cases():
    """render_colorvol (renderer.py:404-407) + render_colorvol_adjoint (:703-709)."""
    rng = np.random.default_rng(31)
    out = {}
    specs = [("a", (7, 8, 6), ((-0.5,) * 3, (0.5,) * 3),
              vd.SphericalCamera(35.0, 20.0, 2.3, fov_y_deg=35.0, width=9, height=8), 0.06),
             ("b", (5, 9, 4), ((-0.4, -0.6, -0.3), (0.6, 0.5, 0.7)),
              vd.SphericalCamera(210.0, -30.0, 2.2, center=np.array([0.1, -0.05, 0.2]),
                                 fov_y_deg=40.0, width=10, height=7), 0.045),
             ("c", (8, 8, 8), ((-0.5,) * 3, (0.5,) * 3),
              vd.SphericalCamera(0.0, 0.0, 0.3, fov_y_deg=60.0, width=6, height=6), 0.05)]
    for key, dims, box, cam, dt in specs:
        vals = np.concatenate([rng.uniform(0.0, 1.0, dims + (3,)),
                               rng.uniform(-0.2, 3.0, dims + (1,))], axis=-1)   # tau < 0 too
        vals = f32(vals)
        cv = vd.ColorVolume(vals, np.array(box[0]), np.array(box[1]))
        seed = f32(rng.normal(size=(cam.height, cam.width, 4)))
        img = vd.render_colorvol(cv, cam, vd.RenderConfig(dt=dt, target="volume")).data
        out[f"{key}_values"] = vals.astype(np.float32)
        out[f"{key}_box"] = np.array(box, np.float64)
        out[f"{key}_cam"] = cam_fields(cam)
        out[f"{key}_dt"] = np.float64(dt)
        out[f"{key}_seed"] = seed
        out[f"{key}_image"] = img
        out[f"{key}_image_none"] = vd.render_colorvol(cv, cam, vd.RenderConfig(dt=dt)).data
        for mode in ("inversion", "stored"):
            gs = vd.render_colorvol_adjoint(
                cv, cam, vd.RenderConfig(dt=dt, target="volume", memory_mode=mode), seed)
            out[f"{key}_{mode}_d_color"] = gs.d_color
    save("color", **out)


def forward_grad_cases():
    """render_forward_grad (renderer.py:410-464) per-pixel Jacobians, camera and stepsize."""
    out = {}
    for s in (500, 501, 502, 2001):
        sc = random_scene(s, tf_res=8 if s != 502 else 2)
        vol, tex = f32(sc.volume.values), f32(sc.tf.texels)
        V, T = vd.DensityVolume(vol), vd.TransferFunction(tex)
        for t in ("camera", "stepsize"):
            img, jac = vd.render_forward_grad(V, T, sc.cam, vd.RenderConfig(dt=sc.dt, target=t))
            out[f"s{s}_{t}_image"] = img.data
            out[f"s{s}_{t}_jac"] = jac
        out[f"s{s}_volume"] = vol.astype(np.float32)
        out[f"s{s}_texels"] = tex.astype(np.float32)
        out[f"s{s}_cam"] = cam_fields(sc.cam)
        out[f"s{s}_dt"] = np.float64(sc.dt)
    # stepsize closed form scene (test_renderer.py:166-175)
    ones = vd.DensityVolume(np.ones((8, 8, 8)))
    T = vd.TransferFunction(f32(np.tile([0.4, 0.4, 0.4, 1.3], (2, 1))))
    cam = vd.SphericalCamera(0.0, 0.0, 2.0, fov_y_deg=8.0, width=9, height=9)
    img, jac = vd.render_forward_grad(ones, T, cam, vd.RenderConfig(dt=0.05, target="stepsize"))
    out["kat_stepsize_jac"] = jac
    save("forward_grad", **out)


def optim_cases():
    """Steps either side of the path: priors, Adam, projection, upsample."""
    from voldiff import objectives as vo
    from voldiff import optim as vopt
    rng = np.random.default_rng(11)
    vol = f32(rng.uniform(-0.2, 1.2, (7, 5, 6)))
    pv, pg = vo.smoothness_prior_volume(vol)
    tex = f32(rng.uniform(-0.5, 3.0, (9, 4)))
    tv, tg = vo.smoothness_prior_tf(vd.TransferFunction(tex))
    grads = [f32(rng.normal(size=vol.shape)) for _ in range(3)]
    st = vopt.OptimState(lr=0.05)
    p = vol.copy()
    traj = []
    for g in grads:
        st, p = vopt.adam_step(st, p, g)
        traj.append(p.copy())
    proj_vol = vopt.project_params(vol, "volume")
    proj_tf = vopt.project_params(tex * 40.0, "tf")
    small = f32(rng.uniform(0, 1, (3, 4, 2)))
    up = vopt.upsample_volume(vd.DensityVolume(small)).values
    save("optim", volume=vol, prior_value=np.float64(pv), prior_grad=pg, texels=tex,
         prior_tf_value=np.float64(tv), prior_tf_grad=tg, adam_grads=np.stack(grads),
         adam_traj=np.stack(traj), adam_lr=np.float64(0.05), proj_vol=proj_vol,
         proj_tf_in=tex * 40.0, proj_tf=proj_tf, up_src=small, up=up)


def entropy_cases():
    """opacity_entropy (objectives.py:95-126) on fp32-representable alpha channels,
    incl. the acceptance contract's images (test_acceptance.py:135-163) and edges."""
    from voldiff import objectives as vo
    rng = np.random.default_rng(13)
    imgs = {}
    u = np.zeros((8, 8, 4)); u[..., 3] = f32(0.42); imgs["uniform"] = u
    o = np.zeros((8, 8, 4)); o[3, 5, 3] = f32(0.9); imgs["onehot"] = o
    r = np.zeros((16, 12, 4)); r[..., 3] = f32(rng.uniform(0.01, 1.0, (16, 12)))
    r[..., :3] = f32(rng.uniform(0, 1, (16, 12, 3))); imgs["random"] = r
    z = r.copy(); z[2:5, 3:9, 3] = 0.0; imgs["zeros"] = z      # p = 0: the +1e6 seed
    imgs["scaled"] = np.where(np.arange(4) == 3, r * np.float32(123.4), r).astype(np.float64)
    imgs["scaled"][..., 3] = f32(imgs["scaled"][..., 3])
    imgs["empty"] = np.zeros((5, 7, 4))                       # degenerate
    imgs["single"] = np.full((1, 1, 4), 0.5)                  # n < 2: degenerate
    n = r.copy(); n[0, 0, 3] = -0.25; imgs["negative"] = n    # a < 0: excluded from F
    out = {}
    for k, im in imgs.items():
        h, seed, deg = vo.opacity_entropy(im)
        out[f"{k}_image"] = im
        out[f"{k}_h"] = np.float64(h)
        out[f"{k}_seed"] = seed
        out[f"{k}_degenerate"] = np.bool_(deg)
    save("entropy", **out)


def io_cases():
    """Files written by the reference's fileio (fileio.py:27-127) + fibonacci_views poses."""
    import json
    from voldiff import fileio as vf
    from voldiff import tasks as vt
    d = os.path.join(OUT, "io")
    os.makedirs(d, exist_ok=True)
    rng = np.random.default_rng(12)
    vol = vd.DensityVolume(f32(rng.uniform(0, 1, (5, 6, 7))), [-1, -2, -3], [1, 2, 3])
    vf.save_volume(vol, os.path.join(d, "vol_a"))
    counts = np.round(rng.uniform(0, 4095, (6, 4, 5))).astype("<f4")
    vf.save_volume(vd.DensityVolume(counts.astype(np.float64) / 4095.0), os.path.join(d, "vol_r"))
    with open(os.path.join(d, "vol_r.raw"), "wb") as fh:
        fh.write(counts.ravel(order="F").tobytes())
    meta = json.load(open(os.path.join(d, "vol_r.json")))
    meta["value_range"] = [100.0, 4095.0]
    with open(os.path.join(d, "vol_r.json"), "w") as fh:
        json.dump(meta, fh)
    vol_r = vf.load_volume(os.path.join(d, "vol_r.raw"))
    tf = vd.TransferFunction(f32(rng.uniform(0, 2, (5, 4))))
    vf.save_tf(tf, os.path.join(d, "tf.json"))
    img = np.zeros((5, 7, 4))
    img[..., 3] = f32(rng.uniform(0, 1, (5, 7)))
    img[..., :3] = f32(img[..., 3:4] * rng.uniform(0, 1.1, (5, 7, 3)))   # some rgb > alpha
    img[0, 0] = 0.0
    img[0, 1] = [1.0, 0.0, 0.0, 1.0]
    img = vr.ImageRGBA(img)
    vf.save_image(img, os.path.join(d, "img.ppm"))
    vf.save_image(img, os.path.join(d, "img.rgba"))
    views = vt.fibonacci_views(13, 2.5, (0.1, 0.0, -0.2), 35.0, 16, 12)
    save("io", vol_a=vol.values, vol_r=vol_r.values, texels=tf.texels, image=img.data,
         fib=np.array([[c.lon_deg, c.lat_deg] for c in views]))


def field_cases():
    """The point-wise field functions (field.py:186-600): trilinear_sample /
    trilinear_gradients on a grid with values outside [0, 1] (both clamps), points
    inside, outside, on faces and exactly on the tolerance band; tf_sample /
    tf_gradients at R = 1, 2, 8 incl. densities outside [0, 1] and on texel
    centres; opacity_from_density incl. the 1 - EPS_ALPHA clamp; camera_from_sphere /
    camera_gradients for three cameras at integer and fractional pixels."""
    from voldiff import field as vfld
    rng = np.random.default_rng(21)
    out = {}
    for name, dims, bmin, bmax in (("a", (6, 5, 7), [-0.5, -0.5, -0.5], [0.5, 0.5, 0.5]),
                                   ("b", (4, 1, 3), [-1.0, 0.25, -2.0], [1.5, 0.75, 1.0])):
        vals = f32(rng.uniform(-0.3, 1.3, dims))
        vol = vd.DensityVolume(vals, bmin, bmax)
        bmin, bmax = np.array(bmin), np.array(bmax)
        ext = bmax - bmin
        pts = bmin + rng.uniform(-0.1, 1.1, (400, 3)) * ext
        faces = bmin + rng.uniform(0, 1, (60, 3)) * ext
        ax = rng.integers(0, 3, 60)
        side = rng.integers(0, 2, 60)
        faces[np.arange(60), ax] = np.where(side, bmax[ax], bmin[ax])
        band = faces.copy()            # just inside / outside the 1e-9 tolerance
        band[np.arange(60), ax] += np.where(side, 1, -1) * np.where(
            np.arange(60) % 2, 0.5e-9, 2e-9) * ext[ax]
        centres = bmin + (np.stack(np.meshgrid(*[np.arange(d) for d in dims], indexing="ij"),
                                   -1).reshape(-1, 3)[:50] + 0.5) * ext / np.array(dims)
        p = np.concatenate([pts, faces, band, centres])
        out[f"vol_{name}"] = vals
        out[f"box_{name}"] = np.stack([bmin, bmax])
        out[f"pts_{name}"] = p
        out[f"value_{name}"] = vd.trilinear_sample(vol, p)
        sp, w, c = vd.trilinear_gradients(vol, p)
        out[f"spatial_{name}"], out[f"weights_{name}"], out[f"corners_{name}"] = sp, w, c
    for R in (1, 2, 8):
        tf = vd.TransferFunction(f32(rng.uniform(-0.5, 3.0, (R, 4))))
        d = np.concatenate([rng.uniform(-0.2, 1.2, 300), (np.arange(R) + 0.5) / R,
                            [0.0, 1.0, -0.0, 0.5 / R, 1 - 0.5 / R]])
        out[f"tf{R}"] = tf.texels
        out[f"d{R}"] = d
        out[f"tfs{R}"] = vd.tf_sample(tf, d)
        sl, tw, ti = vd.tf_gradients(tf, d)
        out[f"slope{R}"], out[f"tw{R}"], out[f"ti{R}"] = sl, tw, ti
    tau = np.concatenate([rng.uniform(-1.0, 50.0, 300), [0.0, 1e6, 13.815510557964274]])
    for k, dt in enumerate((0.05, 1.0)):
        a, dadt = vd.opacity_from_density(tau, dt)
        out[f"alpha{k}"], out[f"dalpha{k}"], out[f"odt{k}"] = a, dadt, np.float64(dt)
    out["tau"] = tau
    cams = [vd.SphericalCamera(30.0, 20.0, 2.0, fov_y_deg=30.0, width=9, height=7),
            vd.SphericalCamera(-117.5, -61.25, 3.5, (0.1, -0.2, 0.3), 47.0, 16, 16),
            vd.SphericalCamera(400.0, 89.5, 1.25, fov_y_deg=8.0, width=5, height=11)]
    for k, cam in enumerate(cams):
        u = np.concatenate([np.repeat(np.arange(cam.width), cam.height),
                            rng.uniform(0, cam.width, 20)])
        v = np.concatenate([np.tile(np.arange(cam.height), cam.width),
                            rng.uniform(0, cam.height, 20)])
        o, dd = vfld.camera_from_sphere(cam, u, v)
        jo, jd = vfld.camera_gradients(cam, u, v)
        out[f"cam{k}"] = np.array([cam.lon_deg, cam.lat_deg, cam.radius, *cam.center,
                                   cam.fov_y_deg, cam.width, cam.height])
        out[f"u{k}"], out[f"v{k}"] = u, v
        out[f"origin{k}"], out[f"dir{k}"], out[f"jo{k}"], out[f"jd{k}"] = o, dd, jo, jd
    save("fields", **out)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    which = sys.argv[1:] or ["kat", "rand", "config", "count", "optim", "fwdgrad", "color", "io",
                             "entropy", "fields"]
    if "fields" in which:
        field_cases()
    if "entropy" in which:
        entropy_cases()
    if "io" in which:
        io_cases()
    if "color" in which:
        color_cases()
    if "optim" in which:
        optim_cases()
    if "fwdgrad" in which:
        forward_grad_cases()
    if "kat" in which:
        kat_cases()
    if "rand" in which:
        random_cases()
    if "config" in which:
        config_cases()
    if "count" in which:
        count_cases()
    if "step" in which:
        step_cases()
    if "tfstep" in which:
        tf_step_cases()
