"""Parity report: measured GPU-vs-reference errors for every golden case (needs a GPU).

    python tests/parity_report.py > profiles/r02_parity.json

Not a test (pytest does not collect it): it prints the numbers the -m gpu
parity tests assert against their bars, so DESIGN.md can quote them.
rel-L2 = ||gpu - ref|| / ||ref||; the reference is voldiff itself (fp64) via
tests/golden/*.npz.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))

import torch  # noqa: E402

from conftest import golden, golden_names, rel_l2  # noqa: E402
from test_gpu_parity import _grads, _setup  # noqa: E402


def main():
    from paper_2107_12672_b200 import raymarch as R
    from paper_2107_12672_b200.scenes import CONFIGS
    dev = torch.device("cuda", 0)
    report = {"bars": {"n_steps": "exact", "image_rel_l2": 1e-5, "grad_rel_l2": 1e-4},
              "cases": {}}
    worst = {}

    def note(case, key, val):
        report["cases"].setdefault(case, {})[key] = val
        worst[key.split("/")[-1]] = max(worst.get(key.split("/")[-1], 0.0), val)

    for name in golden_names("kat_") + golden_names("rand_"):
        g = golden(name)
        for layout in ("cells", "voxels"):
            dens, tex, cams, rig, dt, cells = _setup(g, dev, layout=layout)
            _, n, _ = R.ray_setup(cams, dt, rig, dims=g["volume"].shape)
            report["cases"].setdefault(name, {})["n_steps_exact"] = bool(
                np.array_equal(n[0].cpu().numpy().ravel(), g["n_steps"].ravel()))
            img, depth = R.forward(dens, tex, cams, dt, rig, cells=cells)
            if np.linalg.norm(g["image"]) > 0:
                note(name, f"{layout}/image", rel_l2(img[0].double().cpu().numpy(), g["image"]))
            seed = torch.from_numpy(np.asarray(g["seed"], np.float32)).to(dev)[None].contiguous()
            for t in ("tf", "volume", "camera", "stepsize"):
                key = f"inversion_{t}"
                if key not in g or np.linalg.norm(g[key]) == 0:
                    continue
                got = _grads(dens, tex, cams, rig, dt, img, depth, seed, [t], cells=cells)[t]
                note(name, f"{layout}/d_{t}", rel_l2(got, g[key]))
    for name in ("C1", "C2", "C3", "C4", "C5"):
        g = dict(golden(name))
        c = CONFIGS[name]
        vol = c.volume()
        g["volume"] = vol
        dens, tex, cams, rig, dt, cells = _setup(g, dev, rows=g["rows"], layout="cells")
        _, n, _ = R.ray_setup(cams, dt, rig, dims=vol.shape)
        report["cases"].setdefault(name, {})["n_steps_exact"] = bool(
            np.array_equal(n[0].cpu().numpy().ravel(), g["n_steps"].ravel()))
        img, depth = R.forward(dens, tex, cams, dt, rig, cells=cells)
        note(name, "cells/image", rel_l2(img[0].double().cpu().numpy(), g["image"]))
        seed = torch.from_numpy(g["seed_band"].astype(np.float32)).to(dev)[None].contiguous()
        targets = sorted({k.split("_")[1] for k in g if k.startswith("inversion_")})
        got = _grads(dens, tex, cams, rig, dt, img, depth, seed, targets, cells=cells)
        for t in targets:
            if t == "volume" and "inversion_volume_idx" in g:
                ref = np.zeros(vol.size)
                ref[g["inversion_volume_idx"]] = g["inversion_volume_val"]
            else:
                ref = g[f"inversion_{t}"]
            note(name, f"cells/d_{t}", rel_l2(got[t], ref))
        report["cases"][name]["band_rows"] = [int(r) for r in g["rows"]]
    # the benchmarked fused step at config scale (test_gpu_step_config.py)
    from paper_2107_12672_b200.distributed import ShardedStep
    from test_gpu_step_config import MODES, step_estimate
    for case, tape, skip, split in MODES:
        g = golden(case)
        name, _, kind = case.split("_")
        c = CONFIGS[name]
        est = torch.from_numpy(step_estimate(name, kind).astype(np.float32)).to(dev)
        tex = torch.from_numpy(g["texels"]).to(dev)
        poses = c.view_poses()
        ll = torch.tensor([poses[int(k)] for k in g["views"]], dtype=torch.float64, device=dev)
        r0, r1 = (int(r) for r in g["rows"])
        rig = R.Rig(c.image, c.image, rows=(r0, r1))
        step = ShardedStep(est, tex, ll, torch.from_numpy(g["refs"]).to(dev).contiguous(),
                           float(g["dt"]), rig, total_elements=float(g["count"]),
                           radius=c.radius, fov_y_deg=c.fov, keep_images=True, band_tape=tape,
                           empty_skip=skip, split_walk=split)
        f = step.run()
        want = np.zeros(est.numel())
        want[g["volume_idx"]] = g["volume_val"]
        key = f"{case}/tape={int(step.band_tape)},skip={int(skip)},split={int(split)}"
        note(key, "step/image", rel_l2(step.img.double().cpu().numpy(), g["image"]))
        note(key, "step/loss", abs(float(f.loss) - float(g["loss"])) / float(g["loss"]))
        note(key, "step/d_volume", rel_l2(f.d_volume.double().cpu().numpy(), want))
        report["cases"][key]["band_rows"] = [r0, r1]
        report["cases"][key]["views"] = [int(k) for k in g["views"]]
    for case, split in (("C1_step_dense", "auto"), ("C1_step_dense", 1),
                        ("C2_step_dense", "auto"), ("C2_step_dense", 1)):
        # the fused TF-target steps, with the default ray split (8 lanes per ray on these
        # bands) and one thread per ray
        g = golden(case)
        name = case.split("_")[0]
        c = CONFIGS[name]
        est = torch.from_numpy(step_estimate(name, "dense").astype(np.float32)).to(dev)
        poses = c.view_poses()
        ll = torch.tensor([poses[int(k)] for k in g["views"]], dtype=torch.float64, device=dev)
        r0, r1 = (int(r) for r in g["rows"])
        step = ShardedStep(est, torch.from_numpy(g["texels"]).to(dev), ll,
                           torch.from_numpy(g["refs"]).to(dev).contiguous(), float(g["dt"]),
                           R.Rig(c.image, c.image, rows=(r0, r1)), targets=tuple(c.targets),
                           total_elements=float(g["count"]), radius=c.radius, fov_y_deg=c.fov,
                           keep_images=True, ray_split=split)
        f = step.run()
        key = f"{case}/targets={'+'.join(c.targets)},ray_split={split}"
        note(key, "step/image", rel_l2(step.img.double().cpu().numpy(), g["image"]))
        note(key, "step/loss", abs(float(f.loss) - float(g["loss"])) / float(g["loss"]))
        note(key, "step/d_tf", rel_l2(f.d_tf.double().cpu().numpy().reshape(-1),
                                      g["d_tf"].reshape(-1)))
        if "volume" in c.targets:
            want = np.zeros(est.numel())
            want[g["volume_idx"]] = g["volume_val"]
            note(key, "step/d_volume", rel_l2(f.d_volume.double().cpu().numpy(), want))
        report["cases"][key]["band_rows"] = [r0, r1]
        report["cases"][key]["views"] = [int(k) for k in g["views"]]
    report["worst"] = worst
    print(json.dumps(report, indent=1, sort_keys=True))


if __name__ == "__main__":
    main()
