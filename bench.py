"""Benchmark: KKT refactor+solve ms per IPM iteration (FP64) on synthetic distillation-column iterates.

Contract (driver): python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  * one step = one interior-point iteration of the hot path: condensation,
    numeric Cholesky, HyKKT solve (Schur CG + recovery + Richardson refinement) for the next iterate
    of a synthetic 18-iterate trajectory whose values are resident in HBM;
  * default workload = config 3 (largest PAPER.md instance, N = 50,000: n = 3,350,067), one system
    per GPU; with N GPUs each rank solves its own instance (different initial state) = weak scaling;
  * value = max-over-ranks device time / (steps x ranks)  [ms per IPM iteration, lower is better];
  * e2e = same metric through ckkt_iterate_host (H2D of the step's values + rhs, D2H of the step);
  * --impl reference = the CPU oracle (oracle/), timed on a bounded sample on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (N, batch, description)
    "c1": (50, 1, "distillation column N=50, single KKT system"),
    "c2": (1000, 1, "distillation column N=1000, single KKT system, 18-iterate trajectory"),
    "c3": (50000, 1, "distillation column N=50000 (largest in PAPER.md Table I), single system per GPU"),
    "c4": (1000, 64, "batch of 64 NMPC instances N=1000 sharded over the GPUs"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ckkt", choices=["ckkt", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--leaf", type=int, default=1072)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-lifted", action="store_true")
    return ap.parse_args()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                parts = [p.strip() for p in out.stdout.strip().split(",")]
                if len(parts) >= 7:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower().startswith("active")})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(self.samples[0][1]), "reasons": reasons,
                "samples": len(self.samples)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def build_inputs(N, instances, dev):
    """Values of the 18-iterate trajectories of the given instances, stacked [T, B, len] on `dev`."""
    import numpy as np
    import torch
    from inputs import distillation as dist
    insts = [dist.Instance(N, i) for i in instances]
    trajs = [inst.trajectory() for inst in insts]
    pat = insts[0].model.pat
    n, m = pat.n, pat.m
    T = len(trajs[0])
    rngs = [np.random.default_rng(3000 + i) for i in instances]
    st = lambda f: torch.as_tensor(np.stack([np.stack([getattr(tr[k], f) for tr in trajs]) for k in range(T)]),
                                   device=dev)
    rhs = lambda cols: torch.as_tensor(np.stack([np.stack([r.standard_normal(cols) for r in rngs]) for _ in range(T)]),
                                       device=dev)
    return {"pat": pat, "n": n, "m": m, "B": len(instances),
            "w": st("w_val"), "j": st("j_val"), "sig": st("sigma_x"), "dl": st("d_lifted"),
            "r1": rhs(n), "ra": rhs(m), "rb": rhs(m)}


def run_ckkt(args, world, rank, local):
    import numpy as np
    import torch
    from paper_2403_15913_b200 import ckkt
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", device_id=dev)
    from paper_2403_15913_b200.sharding import max_over_ranks, per_unit_ms, shard
    N, batch, desc = CONFIGS[args.config]
    t0 = time.time()
    # config 4 shards a fixed batch of instances over the ranks (strong scaling); the single-system
    # configs give every rank its own instance (weak scaling)
    mine = list(shard(batch, world, rank)) if batch > 1 else [rank]
    total_units = batch if batch > 1 else world
    data = build_inputs(N, mine, dev)
    pat, n, m, B = data["pat"], data["n"], data["m"], data["B"]
    T = data["w"].shape[0]
    stream = torch.cuda.current_stream()
    t1 = time.time()
    ctx = ckkt.Context(n, m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, strategy=ckkt.CKKT_HYKKT,
                       leaf=args.leaf, batch=B, device=local, stream=stream.cuda_stream)
    setup_s = time.time() - t1
    sizes = ctx.get_sizes()
    dx = torch.empty((B, n), dtype=torch.float64, device=dev)
    dy = torch.empty((B, m), dtype=torch.float64, device=dev)
    notpd = torch.zeros(B, dtype=torch.int32, device=dev)

    def step(k, c=ctx):
        c.refactor(data["w"][k], data["j"][k], None, data["sig"][k], None, None, notpd, None)
        rc, info = c.solve(data["r1"][k], None, data["ra"][k], None, dx, None, dy, None, want_info=True)
        return rc, info

    infos = []
    for k in range(args.warmup):
        step(k % T)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record(stream)
        for k in range(args.steps):
            rc, info = step((args.warmup + k) % T)
            infos.extend(info)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = ctx.launch_count() - l0
    ms = max_over_ranks(ev0.elapsed_time(ev1), dev)
    # phase split for the roofline: a second timed pass of the same steps with CUDA events around every
    # condense / factor / forward / backward / vector launch group (event brackets cannot live inside the
    # CG graph, so this pass runs the host-driven CG loop; kernel durations are the same)
    prof_steps = min(args.steps, 3)
    ctx.profile(True)
    for k in range(prof_steps):
        step((args.warmup + k) % T)
    phases = ctx.phase_times()
    ctx.profile(False)
    phases = {k: (v[0] * args.steps / prof_steps, v[1] * args.steps / prof_steps) for k, v in phases.items()}
    # Lifted-KKT on the same instance (extra key)
    lifted = None
    if not args.no_lifted:
        ctxl = ckkt.Context(n, 0, m, pat.w_row, pat.w_col, None, None, pat.j_rowptr, pat.j_col,
                            strategy=ckkt.CKKT_LIFTED, leaf=args.leaf, batch=B, device=local,
                            stream=stream.cuda_stream)
        ds = torch.empty((B, m), dtype=torch.float64, device=dev)
        dz = torch.empty((B, m), dtype=torch.float64, device=dev)

        def lstep(k):
            ctxl.refactor(data["w"][k], None, data["j"][k], data["sig"][k], data["dl"][k], None, notpd, None)
            return ctxl.solve(data["r1"][k], data["ra"][k], None, data["rb"][k], dx, ds, None, dz)

        for k in range(args.warmup):
            lstep(k % T)
        torch.cuda.synchronize()
        linfo = []
        ev0.record(stream)
        for k in range(args.steps):
            linfo.extend(lstep((args.warmup + k) % T)[1])
        ev1.record(stream)
        torch.cuda.synchronize()
        lifted = {"ms_per_iter": per_unit_ms(max_over_ranks(ev0.elapsed_time(ev1), dev), args.steps, total_units),
                  "n_ref_mean": float(np.mean([i["n_ref"] for i in linfo])),
                  "rel_res_max": float(max(i["rel_res"] for i in linfo)),
                  "rel_res_unrefined_max": float(max(i["rel_res_unrefined"] for i in linfo)),
                  "status_max": int(max(i["status"] for i in linfo))}
        ctxl.close()
    # e2e through the public host API (pinned host buffers)
    e2e = None
    if not args.no_e2e:
        hw = data["w"].cpu().pin_memory()
        hj = data["j"].cpu().pin_memory()
        hs = data["sig"].cpu().pin_memory()
        hr1 = data["r1"].cpu().pin_memory()
        hra = data["ra"].cpu().pin_memory()
        hdx = torch.empty((B, n), dtype=torch.float64).pin_memory()
        hdy = torch.empty((B, m), dtype=torch.float64).pin_memory()
        for k in range(args.warmup):
            ctx.iterate_host(hw[k], hj[k], None, hs[k], None, None, hr1[k], None, hra[k], None, hdx, None, hdy, None)
        torch.cuda.synchronize()
        ev0.record(stream)
        for k in range(args.steps):
            kk = (args.warmup + k) % T
            ctx.iterate_host(hw[kk], hj[kk], None, hs[kk], None, None, hr1[kk], None, hra[kk], None, hdx, None, hdy,
                             None)
        ev1.record(stream)
        torch.cuda.synchronize()
        e_ms = max_over_ranks(ev0.elapsed_time(ev1), dev)
        h2d = 8 * B * (hw.shape[-1] + hj.shape[-1] + hs.shape[-1] + hr1.shape[-1] + hra.shape[-1])
        d2h = 8 * B * (n + m)
        e2e = {"value": per_unit_ms(e_ms, args.steps, total_units), "unit": "ms/IPM-iter",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    # roofline of the dominant kernel phase: algorithmic bytes per launch
    #   forward / backward sweep: read every panel once + read/write x   = 8 (l_storage + 2 n)
    #   factorization:            read K, write L                        = 8 (nnz_k + l_storage)
    #   condensation:             read W, J, Sigma, maps; write K
    algo = {"forward": 8.0 * B * (sizes["l_storage"] + 2 * n), "backward": 8.0 * B * (sizes["l_storage"] + 2 * n),
            "factor": 8.0 * B * (sizes["nnz_k"] + sizes["l_storage"]),
            "condense": 8.0 * B * (len(pat.w_row) + len(pat.j_col) + n + sizes["nnz_k"])}
    dom = max((k for k in phases if k in algo), key=lambda k: phases[k][0])
    dom_ms, dom_n = phases[dom]
    avg = dom_ms / max(dom_n, 1)
    achieved = algo[dom] / (avg * 1e-3) / 1e9
    peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)" if "when" in peaks else "fallback"
    roof = {"bound": "hbm", "kernel": {"forward": "k_fwd_tiny + k_fwd_persist + k_fwd_top (one forward sweep)",
                                       "backward": "k_bwd_top + k_bwd_persist + k_bwd_tiny (one backward sweep)",
                                       "factor": "k_factor_persist", "condense": "k_condense"}[dom],
            "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
            "traffic": None, "peak_source": peak_src, "algorithmic_bytes_per_launch": algo[dom],
            "avg_launch_ms": avg,
            "phase_pass": "CUDA events per launch group, separate timed pass of min(steps, 3) steps of the same workload",
            "phases_ms_per_step": {k: v[0] / args.steps for k, v in phases.items()},
            "launches_per_step": {k: v[1] / args.steps for k, v in phases.items()}}
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tr_path):  # DRAM bytes per launch of this kernel from the committed ncu capture
        roof["traffic"] = json.load(open(tr_path)).get(roof["kernel"])
    fac_ms = phases["factor"][0] / max(phases["factor"][1], 1)
    fp64 = {"kernel": "k_factor_persist", "flops": B * sizes["flops_factor"], "ms": fac_ms,
            "achieved_tflops": B * sizes["flops_factor"] / (fac_ms * 1e-3) / 1e12, "peak_tflops": 37.1,
            "peak_source": "measured DFMA/DMMA microbenchmark, profiles/fp64_peak_r01.txt"}
    fp64["frac"] = fp64["achieved_tflops"] / fp64["peak_tflops"]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(data, args)
    info_summary = {"k_cg_mean": float(np.mean([i["k_cg"] for i in infos])),
                    "rel_res_unrefined_max": float(max(i["rel_res_unrefined"] for i in infos)),
                    "n_ref_mean": float(np.mean([i["n_ref"] for i in infos])),
                    "rel_res_max": float(max(i["rel_res"] for i in infos)),
                    "status_max": int(max(i["status"] for i in infos))}
    out = {
        "metric": "KKT refactor+solve ms/IPM-iter (FP64)",
        "value": per_unit_ms(ms, args.steps, total_units),
        "unit": "ms/IPM-iter",
        "higher_is_better": False,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps,
        "scaling": "strong" if batch > 1 else "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic distillation-column IPM iterates (inputs/distillation.py), random N(0,1) rhs",
        "config": {"workload": desc, "N": N, "n": n, "m_e": m, "strategy": "HyKKT gamma=1e7",
                   "instances_per_gpu": B, "units": "one IPM iteration of one KKT system",
                   "leaf": args.leaf, "l2": "inputs larger than L2 (L factor %.2f GB)" % (sizes["l_storage"] * 8 / 1e9),
                   "parallelism": f"replicas x{world}"},
        "phases_ms": {"refactor": (phases["condense"][0] + phases["factor"][0]) / args.steps,
                      "sweeps": (phases["forward"][0] + phases["backward"][0]) / args.steps,
                      "vector": phases["vector"][0] / args.steps,
                      "other": ms / args.steps - sum(v[0] for v in phases.values()) / args.steps},
        "solver": info_summary,
        "lifted": lifted,
        "sizes": sizes,
        "setup_s": setup_s,
        "gen_s": t1 - t0,
        "roofline": roof,
        "factor_fp64": fp64,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline(data, args, N_sample=10000):
    """The oracle as it stands, single-threaded, one HyKKT IPM iteration (refactor + solve) on a
    bounded sample: the same model at N_sample stages, scaled to N by the stage count (work per stage
    is constant for the nested-dissection ordering)."""
    import numpy as np
    from inputs import distillation as dist
    from oracle import kkt as OK
    N = CONFIGS[args.config][0]
    Ns = min(N, N_sample)
    inst = dist.Instance(Ns, 0)
    it = inst.iterate(9, 1.5e-4)
    pat = inst.model.pat
    e32 = np.zeros(1, np.int32)
    o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, e32, e32[:0], leaf=args.leaf)
    rng = np.random.default_rng(1)
    t = time.perf_counter()
    o.refactor(it.w_val, it.j_val, np.zeros(0), it.sigma_x, np.zeros(0), 0.0)
    d, info = o.solve(rng.standard_normal(pat.n), np.zeros(0), rng.standard_normal(pat.m), np.zeros(0))
    el = time.perf_counter() - t
    return {"value": el * 1e3 * (N / Ns), "unit": "ms/IPM-iter", "cores": 1, "kind": "oracle",
            "sample": f"one HyKKT iteration (refactor+solve, k_cg={info.k_cg}, n_ref={info.n_ref}) at N={Ns}, "
                      f"scaled x{N / Ns:g} to N={N}; measured {el:.1f} s"}


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle as it stands, on rank 0 only."""
    if rank != 0:
        return
    import numpy as np
    from inputs import distillation as dist
    from oracle import kkt as OK
    N = CONFIGS[args.config][0]
    Ns = min(N, 2000)
    inst = dist.Instance(Ns, 0)
    traj = inst.trajectory()
    pat = inst.model.pat
    e32 = np.zeros(1, np.int32)
    o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, e32, e32[:0], leaf=args.leaf)
    rng = np.random.default_rng(1)

    def step(k):
        it = traj[k % len(traj)]
        o.refactor(it.w_val, it.j_val, np.zeros(0), it.sigma_x, np.zeros(0), 0.0)
        return o.solve(rng.standard_normal(pat.n), np.zeros(0), rng.standard_normal(pat.m), np.zeros(0))

    for k in range(args.warmup):
        step(k)
    t = time.perf_counter()
    for k in range(args.steps):
        step(args.warmup + k)
    el = time.perf_counter() - t
    v = el * 1e3 / args.steps * (N / Ns)
    sample = f"oracle HyKKT iterations (refactor+solve) at N={Ns}, scaled x{N / Ns:g} to N={N}"
    print(json.dumps({
        "impl": "reference", "metric": "KKT refactor+solve ms/IPM-iter (FP64)", "value": v, "unit": "ms/IPM-iter",
        "higher_is_better": False, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": v, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic distillation-column IPM iterates", "config": {"workload": CONFIGS[args.config][2], "N": N},
        "cpu_baseline": {"value": v, "unit": "ms/IPM-iter", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "ms/IPM-iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def main():
    args = parse()
    world, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ckkt(args, world, rank, local)


if __name__ == "__main__":
    main()
