"""Benchmark: KKT refactor+solve ms per IPM iteration (FP64) on synthetic distillation-column iterates.

Contract (driver): python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  * one step = one interior-point iteration of the hot path: condensation,
    numeric Cholesky, HyKKT solve (Schur CG + recovery + Richardson refinement) for the next iterate
    of a synthetic 18-iterate trajectory whose values are resident in HBM;
  * default workload = config 3 (largest PAPER.md instance, N = 50,000: n = 3,350,067), one system
    per GPU; with N GPUs each rank solves its own instance (different initial state) = weak scaling;
  * value = max-over-ranks device time / (steps x ranks)  [ms per IPM iteration, lower is better];
  * e2e = same metric through ckkt_iterate_host (H2D of the step's values + rhs, D2H of the step);
  * --impl reference = the CPU oracle (oracle/) as it stands, single-threaded, at the same workload and
    iterates on rank 0 (min(warmup, 1) untimed + min(steps, 3) timed iterations, median);
  * --gpus N without WORLD_SIZE in the environment re-executes itself under torchrun (N ranks).
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


def trajectory_rhs(n, m, instance, T):
    """The seeded right-hand sides of one instance's trajectory: r1 [T, n], then r3 (or r2) [T, m], then
    r4 [T, m], drawn in that order from the generator 3000 + instance (one stream shared by both arms)."""
    import numpy as np
    rng = np.random.default_rng(3000 + instance)
    r1 = np.stack([rng.standard_normal(n) for _ in range(T)])
    ra = np.stack([rng.standard_normal(m) for _ in range(T)])
    rb = np.stack([rng.standard_normal(m) for _ in range(T)])
    return r1, ra, rb


def trajectory_positions(inst, ks, per_mu=3):
    """Iterates at trajectory positions ks (Instance.trajectory()[k] without building the others)."""
    from inputs import distillation as dist
    mus = dist.mu_schedule()
    return {k: inst.iterate(k, mus[k // per_mu]) for k in ks}


def trajectory_length(per_mu=3):
    from inputs import distillation as dist
    return per_mu * len(dist.mu_schedule())


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
    assert T == trajectory_length()
    st = lambda f: torch.as_tensor(np.stack([np.stack([getattr(tr[k], f) for tr in trajs]) for k in range(T)]),
                                   device=dev)
    rh = [trajectory_rhs(n, m, i, T) for i in instances]
    rhs = lambda j: torch.as_tensor(np.stack([r[j] for r in rh], axis=1), device=dev)  # [T, B, len]
    it0 = trajs[0][0]
    return {"pat": pat, "n": n, "m": m, "B": len(instances),
            "w": st("w_val"), "j": st("j_val"), "sig": st("sigma_x"), "dl": st("d_lifted"),
            "r1": rhs(0), "ra": rhs(1), "rb": rhs(2),
            "model": (insts[0].model, insts[0].xbar0, it0.v, it0.lam, insts[0].row_scale, insts[0].obj_scale)}


def bench_config(args, world, n, m):
    """The workload description shared by both arms (same_config)."""
    N, batch, desc = CONFIGS[args.config]
    large = N * 67 * 47 * 8 * max(batch, 1) > 126e6  # L factor ~47 doubles per variable (ND, leaf 1072)
    return {"workload": desc, "N": N, "n": n, "m_e": m, "strategy": "HyKKT gamma=1e7",
            "instances": batch if batch > 1 else world, "units": "one IPM iteration of one KKT system",
            "leaf": args.leaf,
            "l2": ("inputs larger than L2 (factor > 126 MB L2 per GPU); no flush" if large else
                   "factor L2-resident (< 126 MB); no flush, repeated solves hit L2"),
            "parallelism": (f"batch sharded over {world} GPU(s), no collective" if batch > 1
                            else f"replicas x{world} (one instance per GPU, no collective)")}


def host_info():
    import platform
    model = platform.processor()
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


def oracle_iterations(N, instance, ks, leaf, warmup=1):
    """The oracle as it stands (oracle/kkt.py + oracle/csrc), single-threaded (BLAS pools limited to one
    thread), one HyKKT IPM iteration = refactor + solve per trajectory position in ks, after `warmup`
    untimed iterations on the first position.  Returns per-iteration seconds and the last Info."""
    import numpy as np
    from threadpoolctl import threadpool_limits
    from inputs import distillation as dist
    from oracle import kkt as OK
    inst = dist.Instance(N, instance)
    its = trajectory_positions(inst, sorted(set(ks)))
    pat = inst.model.pat
    T = trajectory_length()
    r1, ra, _ = trajectory_rhs(pat.n, pat.m, instance, T)
    e32 = np.zeros(1, np.int32)
    times, info = [], None
    with threadpool_limits(limits=1):
        t = time.perf_counter()
        o = OK.SparseKKT(pat.n, pat.m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, e32, e32[:0], leaf=leaf)
        setup_s = time.perf_counter() - t
        for j, k in enumerate([ks[0]] * warmup + list(ks)):
            it = its[k]
            t = time.perf_counter()
            o.refactor(it.w_val, it.j_val, np.zeros(0), it.sigma_x, np.zeros(0), 0.0)
            d, info = o.solve(r1[k], np.zeros(0), ra[k], np.zeros(0))
            if j >= warmup:
                times.append(time.perf_counter() - t)
    return times, info, setup_s


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
    # NEXT-2: the analysis exported once and reused by a second context
    t2 = time.time()
    blob = ctx.export_analysis()
    export_s = time.time() - t2
    t2 = time.time()
    ckkt.Context(n, m, 0, pat.w_row, pat.w_col, pat.j_rowptr, pat.j_col, None, None, strategy=ckkt.CKKT_HYKKT,
                 leaf=args.leaf, batch=B, device=local, stream=stream.cuda_stream, analysis=blob).close()
    setup_blob_s = time.time() - t2
    blob_bytes = int(blob.size)
    del blob
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
    prof_steps = args.steps  # the same trajectory positions as the timed steps (their n_ref / k_cg differ)
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
    # NEXT-4: the model evaluation of one iterate (J, W, c, grad f) on the GPU (ckkt_distillation_eval) vs
    # the numpy generator on the host (context: the paper's "AD" column)
    md, xbar0, v0, lam0, rs0, sf0 = data["model"]
    Td = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    mv = [Td(xbar0), Td(v0), Td(lam0), Td(rs0)]
    mo = [torch.empty(len(pat.j_col), dtype=torch.float64, device=dev),
          torch.empty(len(pat.w_row), dtype=torch.float64, device=dev),
          torch.empty(m, dtype=torch.float64, device=dev), torch.empty(n, dtype=torch.float64, device=dev)]
    for _ in range(3):
        ckkt.distillation_eval(N, md.p, mv[0], mv[1], mv[2], mv[3], sf0, *mo)
    ev0.record(stream)
    for _ in range(10):
        ckkt.distillation_eval(N, md.p, mv[0], mv[1], mv[2], mv[3], sf0, *mo)
    ev1.record(stream)
    torch.cuda.synchronize()
    me_gpu = ev0.elapsed_time(ev1) / 10
    th = time.perf_counter()
    md.jacobian_values(v0)
    md.hessian_values(v0, lam0 * rs0, sf0)
    md.residual(v0, xbar0)
    md.grad_f(v0)
    model_eval = {"gpu_ms": me_gpu, "host_numpy_ms": (time.perf_counter() - th) * 1e3,
                  "outputs": "J, W (Lagrangian Hessian), c, grad f of one iterate",
                  "bytes": 8 * (len(pat.j_col) + len(pat.w_row) + 2 * m + 2 * n)}
    del mv, mo
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 7700.0}
    peak_src = ("measured (MEASURED_PEAKS.json hbm_gbs)" if "when" in peaks
                else "fallback (B200_PROFILING.md nominal HBM3e)")
    # algorithmic bytes per launch, from the EXACT factor (nnz_l, no amalgamation padding):
    #   forward / backward sweep: read every L entry once + read and write x   = 8 (nnz_l + 2 n)
    #   factorization:            read K, write L                              = 8 (nnz_k + nnz_l)
    #   condensation:             read W, J, Sigma; write K (maps excluded)    = 8 (nnz_w + nnz_j + n + nnz_k)
    nnz_l = sizes["nnz_l"]
    algo = {"forward": 8.0 * B * (nnz_l + 2 * n), "backward": 8.0 * B * (nnz_l + 2 * n),
            "factor": 8.0 * B * (sizes["nnz_k"] + nnz_l),
            "condense": 8.0 * B * (len(pat.w_row) + len(pat.j_col) + n + sizes["nnz_k"])}
    kname = {"forward": "k_fwd_tiny + k_fwd_persist + k_fwd_top (one forward sweep)",
             "backward": "k_bwd_top + k_bwd_persist + k_bwd_tiny (one backward sweep)",
             "factor": "k_factor_tiny + k_factor_persist (one numeric factorization)",
             "condense": "k_condense"}
    # DRAM bytes per launch from the committed ncu capture, which is of the default workload (C3) only
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tr_path)) if os.path.exists(tr_path) and args.config == "c3" else {}

    def roof_entry(ph):
        ms_tot, cnt = phases[ph]
        avg = ms_tot / max(cnt, 1)
        ach = algo[ph] / (avg * 1e-3) / 1e9
        return {"bound": "hbm", "kernel": kname[ph], "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "traffic": traffic.get(kname[ph]), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": algo[ph], "avg_launch_ms": avg,
                "share_of_step": ms_tot / max(sum(v[0] for v in phases.values()), 1e-30)}

    dom = max((k for k in phases if k in algo), key=lambda k: phases[k][0])
    roof = roof_entry(dom)
    roof["phase_pass"] = ("CUDA events on the library stream per launch group, separate pass of the same "
                          "steps of the same workload (host-driven CG loop)")
    roof["phases_ms_per_step"] = {k: v[0] / args.steps for k, v in phases.items()}
    roof["launches_per_step"] = {k: v[1] / args.steps for k, v in phases.items()}
    roof["per_phase"] = {ph: {k: v for k, v in roof_entry(ph).items() if k in ("achieved", "frac", "avg_launch_ms",
                                                                          "traffic", "share_of_step")}
                         for ph in algo}
    # the factorization against the FP64 pipe: algorithmic flops sum_j colcount_j^2 (exact pattern)
    fac_ms = phases["factor"][0] / max(phases["factor"][1], 1)
    fp64 = {"bound": "fp64", "kernel": kname["factor"], "flops_per_launch": B * sizes["flops_factor"],
            "ms": fac_ms, "achieved": B * sizes["flops_factor"] / (fac_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
            "peak": 37.1, "peak_source": "measured FP64 DFMA/DMMA microbenchmark on this B200 pool "
                                         "(profiles/fp64_peak_r01.txt; DMMA m8n8k4 on sm_100a = DFMA rate)"}
    fp64["frac"] = fp64["achieved"] / fp64["peak"]
    fp64["hbm"] = roof["per_phase"]["factor"]
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(args, N, (args.warmup % T))
    info_summary = {"k_cg_mean": float(np.mean([i["k_cg"] for i in infos])),
                    "rel_res_unrefined_max": float(max(i["rel_res_unrefined"] for i in infos)),
                    "n_ref_mean": float(np.mean([i["n_ref"] for i in infos])),
                    "rel_res_max": float(max(i["rel_res"] for i in infos)),
                    "status_max": int(max(i["status"] for i in infos)),
                    # per timed step (instance 0): correction passes and CG iterations, the work that
                    # moves the step time besides the kernels
                    "n_ref_per_step": [int(i["n_ref"]) for i in infos[::B]],
                    "k_cg_total_per_step": [int(i["k_cg_total"]) for i in infos[::B]]}
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
        "data": "synthetic distillation-column IPM iterates (inputs/distillation.py), seeded N(0,1) rhs",
        "config": bench_config(args, world, n, m),
        "phases_ms": {"refactor": (phases["condense"][0] + phases["factor"][0]) / args.steps,
                      "sweeps": (phases["forward"][0] + phases["backward"][0]) / args.steps,
                      "vector": phases["vector"][0] / args.steps,
                      "other": ms / args.steps - sum(v[0] for v in phases.values()) / args.steps},
        "solver": info_summary,
        "lifted": lifted,
        "sizes": sizes,
        "setup_s": setup_s,
        "setup_from_analysis_s": setup_blob_s,
        "analysis_blob": {"bytes": blob_bytes, "export_s": export_s, "threads": os.cpu_count()},
        "gen_s": t1 - t0,
        "roofline": roof,
        "factor_fp64": fp64,
        "e2e": e2e,
        "model_eval": model_eval,
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


def cpu_baseline(args, N, k0):
    """The oracle as it stands, single-threaded, at the bench's own workload: one HyKKT IPM iteration
    (refactor + solve) of instance 0 at trajectory position k0 (the first timed GPU step's iterate and
    rhs), full size.  The oracle has no caches to warm, so the one iteration is timed directly."""
    times, info, setup_s = oracle_iterations(N, 0, [k0], args.leaf, warmup=0)
    return {"value": times[0] * 1e3, "unit": "ms/IPM-iter", "cores": 1, "kind": "oracle",
            "sample": f"one oracle HyKKT iteration (refactor+solve, k_cg={info.k_cg}, n_ref={info.n_ref}) at the "
                      f"full workload N={N}, trajectory position {k0}; BLAS pools limited to 1 thread; oracle "
                      f"setup {setup_s:.0f} s excluded (like the GPU setup)", **host_info()}


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle as it stands, on rank 0 only, at the same workload and iterates as
    the GPU arm (instance 0, trajectory positions warmup + k): min(warmup, 1) untimed and min(steps, 3)
    timed iterations, median."""
    if rank != 0:
        return
    import numpy as np
    N = CONFIGS[args.config][0]
    T = trajectory_length()
    wu, ks = min(args.warmup, 1), [(args.warmup + k) % T for k in range(min(args.steps, 3))]
    times, info, setup_s = oracle_iterations(N, 0, ks, args.leaf, warmup=wu)
    v = float(np.median(times)) * 1e3
    from inputs import distillation as dist
    n, m = dist.dimensions(N)
    sample = (f"{len(times)} oracle HyKKT iterations (refactor+solve) at the full workload N={N}, trajectory "
              f"positions {ks} (the GPU arm's first timed iterates), after {wu} untimed; median; BLAS pools "
              f"limited to 1 thread; per-iteration s = {[float(f"{t:.3g}") for t in times]}; oracle setup "
              f"{setup_s:.0f} s excluded")
    print(json.dumps({
        "impl": "reference", "metric": "KKT refactor+solve ms/IPM-iter (FP64)", "value": v, "unit": "ms/IPM-iter",
        "higher_is_better": False, "n_gpus": world, "steps": len(times), "steps_requested": args.steps,
        "warmup": wu, "ms_per_step": v, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic distillation-column IPM iterates (inputs/distillation.py), seeded N(0,1) rhs",
        "config": bench_config(args, world, n, m),
        "cpu_baseline": {"value": v, "unit": "ms/IPM-iter", "cores": 1, "kind": "oracle", "sample": sample,
                         **host_info()},
        "e2e": {"value": v, "unit": "ms/IPM-iter", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # `python bench.py --gpus N` without a launcher: re-exec under torchrun, one rank per GPU (127.0.0.1
        # rendezvous); rank 0 prints the single JSON line
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)
    world, rank, local = dist_init()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    run_ckkt(args, world, rank, local)


if __name__ == "__main__":
    main()
