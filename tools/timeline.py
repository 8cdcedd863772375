"""Kernel timeline of bench.py's HyKKT step (CUPTI via torch.profiler): busy time vs idle gaps between
consecutive kernels, the largest gap classes by (previous kernel -> next kernel), and per-kernel busy
time.  Explains the "other" share of bench.py's phase split (step time not covered by kernel work).
Usage: python tools/timeline.py [config] [steps]"""
import collections
import json
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2403_15913_b200 import ckkt  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
N, batch, _ = bench.CONFIGS[cfg]
dev = torch.device("cuda:0")
data = bench.build_inputs(N, list(range(batch)) if batch > 1 else [0], dev)
pat, n, m, B = data["pat"], data["n"], data["m"], data["B"]
T = data["w"].shape[0]
stream = torch.cuda.current_stream()
ctx = ckkt.Context(n, m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, strategy=ckkt.CKKT_HYKKT,
                   leaf=1072, batch=B, device=0, stream=stream.cuda_stream)
dx = torch.empty((B, n), dtype=torch.float64, device=dev)
dy = torch.empty((B, m), dtype=torch.float64, device=dev)
notpd = torch.zeros(B, dtype=torch.int32, device=dev)


def step(k):
    ctx.refactor(data["w"][k], data["j"][k], None, data["sig"][k], None, None, notpd, None)
    return ctx.solve(data["r1"][k], None, data["ra"][k], None, dx, None, dy, None, want_info=True)


for k in range(3):
    step(k % T)
torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    ev0.record(stream)
    for k in range(steps):
        step((3 + k) % T)
    ev1.record(stream)
    torch.cuda.synchronize()
wall = ev0.elapsed_time(ev1) * 1e3  # us
# kernel / memcpy / memset records from the chrome trace (names included for kernels launched by libckkt)
with tempfile.NamedTemporaryFile(suffix=".json") as tf:
    prof.export_chrome_trace(tf.name)
    trace = json.load(open(tf.name))
ks = sorted(((float(e["ts"]), float(e["ts"]) + float(e.get("dur", 0.0)), e.get("name", ""))
             for e in trace.get("traceEvents", [])
             if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")), key=lambda t: t[0])
busy, gaps, prev_end, prev_name = 0.0, collections.Counter(), None, None
gapn = collections.Counter()
per = collections.Counter()
cnt = collections.Counter()
for s, e, name in ks:
    short = name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    per[short] += e - s
    cnt[short] += 1
    if prev_end is not None:
        g = s - prev_end
        if g > 0:
            gaps[(prev_name, short)] += g
            gapn[(prev_name, short)] += 1
    busy += max(0.0, e - max(s, prev_end)) if prev_end is not None else e - s
    if prev_end is None or e > prev_end:
        prev_end, prev_name = e, short
tot_gap = sum(gaps.values())
print(f"{cfg}: {steps} steps, event-timed {wall / steps / 1e3:.2f} ms/step, kernel busy {busy / steps / 1e3:.2f} "
      f"ms/step, idle gaps {tot_gap / steps / 1e3:.2f} ms/step over {sum(gapn.values()) / steps:.0f} boundaries/step, "
      f"{len(ks) / steps:.0f} kernels/step")
print("largest gap classes (us per step, count per step, mean us):")
for (a, b), g in gaps.most_common(25):
    print(f"  {g / steps:9.1f} {gapn[(a, b)] / steps:6.1f} {g / gapn[(a, b)]:7.2f}  {a} -> {b}")
print("kernel busy time (us per step, launches per step, mean us):")
for k, v in per.most_common(40):
    print(f"  {v / steps:9.1f} {cnt[k] / steps:6.1f} {v / cnt[k]:8.2f}  {k}")

# the phase split bench.py reports, for the same steps (host-driven CG loop, CUDA events per launch group)
ctx.profile(True)
for k in range(steps):
    step((3 + k) % T)
ph = ctx.phase_times()
ctx.profile(False)
print("phase split of the same steps (ms per step):", {k: round(v[0] / steps, 3) for k, v in ph.items()},
      "sum %.2f" % (sum(v[0] for v in ph.values()) / steps))
