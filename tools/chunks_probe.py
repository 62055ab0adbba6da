"""e2e of the C4 step vs the number of view chunks used to stage the host refs.

    python tools/chunks_probe.py      # GPU
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2107_12672_b200 import raymarch as R                     # noqa: E402
from paper_2107_12672_b200.distributed import ShardedStep, TomographyIteration  # noqa: E402
from paper_2107_12672_b200.scenes import CONFIGS                     # noqa: E402

dev = torch.device("cuda")
cfg = CONFIGS["C4"]
truth = torch.from_numpy(cfg.volume()).to(dev)
tex = torch.from_numpy(cfg.texels().astype(np.float32)).to(dev)
ll = torch.tensor(cfg.view_poses(), dtype=torch.float64, device=dev)
cams = R.camera_array(ll, cfg.radius, (0.0, 0.0, 0.0), cfg.fov)
rig = R.Rig(512, 512)
refs, _ = R.forward(truth, tex, cams, cfg.dt, rig, with_depth=False, cells=R.pack_cells(truth))
est = (0.85 * truth + 0.05).contiguous()
host_vol = est.cpu().pin_memory()
host_refs = refs.cpu().pin_memory()
host_out = torch.empty_like(host_vol).pin_memory()
for chunks in (1, 2, 4, 8, 16):
    step = ShardedStep(est, tex, ll, refs, cfg.dt, rig, total_elements=refs.numel(),
                       chunks=chunks)
    it = TomographyIteration(step)
    ms = []
    for k in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        est.copy_(host_vol, non_blocking=True)
        it.run(refs_host=host_refs)
        host_out.copy_(est, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(a.elapsed_time(b))
    print(f"chunks {chunks:2d}: e2e {np.mean(ms):7.2f} ms/step")
