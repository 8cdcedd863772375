"""Time ckkt_refactor (and one HyKKT solve) at size N with CUDA events; A/B experiments with
CKKT_LIB_OVERRIDE / CKKT_* switches.  Caches the generated iterate under /tmp within one gpurun call.
Usage: python tools/time_refactor.py N [reps] [tag]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from inputs import distillation as dist  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

N = int(sys.argv[1])
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
tag = sys.argv[3] if len(sys.argv) > 3 else os.environ.get("CKKT_LIB_OVERRIDE", "default")
cache = f"/tmp/ckkt_iter_{N}.npz"
pat = dist.build_pattern(N)
if os.path.exists(cache):
    z = np.load(cache)
    w_val, j_val, sig = z["w"], z["j"], z["s"]
else:
    it = dist.Instance(N).iterate(9, 1.5e-4)
    w_val, j_val, sig = it.w_val, it.j_val, it.sigma_x
    np.savez(cache, w=w_val, j=j_val, s=sig)
dev = torch.device("cuda:0")
st = torch.cuda.current_stream()
t = time.time()
ctx = ckkt.Context(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, leaf=1072, device=0,
                   stream=st.cuda_stream)
setup = time.time() - t
v = [torch.as_tensor(a, device=dev) for a in (w_val, j_val, sig)]
rng = np.random.default_rng(3000)
r1 = torch.as_tensor(rng.standard_normal(pat.n), device=dev)
r3 = torch.as_tensor(rng.standard_normal(pat.m), device=dev)
dx = torch.empty(pat.n, dtype=torch.float64, device=dev)
dy = torch.empty(pat.m, dtype=torch.float64, device=dev)
ctx.refactor(v[0], v[1], None, v[2])
rc, info = ctx.solve(r1, None, r3, None, dx, None, dy, None)
ctx.profile(True)
for r in range(reps):
    ctx.refactor(v[0], v[1], None, v[2])
ph = ctx.phase_times()
ctx.solve(r1, None, r3, None, dx, None, dy, None)
ph2 = ctx.phase_times()
ctx.profile(False)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for r in range(reps):
    ctx.refactor(v[0], v[1], None, v[2])
    ctx.solve(r1, None, r3, None, dx, None, dy, None, want_info=False)
e1.record(st)
torch.cuda.synchronize()
fw = ph2["forward"]
bw = ph2["backward"]
print(f"[{tag}] N={N} factor {ph['factor'][0] / reps:.3f} ms  condense {ph['condense'][0] / reps:.3f} ms  "
      f"fwd sweep {fw[0] / max(fw[1], 1):.3f} ms  bwd sweep {bw[0] / max(bw[1], 1):.3f} ms  "
      f"iter {e0.elapsed_time(e1) / reps:.2f} ms  k_cg {info[0]['k_cg']} n_ref {info[0]['n_ref']} "
      f"rel_res {info[0]['rel_res']:.2e} setup {setup:.1f} s", flush=True)
