"""Benchmark: implicit-Euler HODLR time-steps/s on BASELINE.json's n = 65536 1D workload (cfg3).

One "step" = one pass of the hot path over one time level with new
d+-(x, t_m) every step: assembly of the diagonally scaled HODLR of A_m (S3), leaf LU +
Sherman-Morrison-Woodbury factorisation (S4-S5), tree solve (S6, fused as an extra right-hand-
side column) and rhs formation u + dt f (S7).  The headline times `--steps` consecutive time
levels through the C-ABI fde1d_run: ONE persistent launch (k_run) in which the leaf work of
step m+1 (which does not depend on u^(m)) runs under the latency-bound tree levels of step m.
The GL weights (S1) and the compression of T_alpha (S2) depend on (alpha, n, leaf, tol) only
-- T is the same matrix at every step and the paper builds A_m's HODLR from it by diagonal
scaling and shift -- so they run once when the handle is built.  Also reported
(other_variant): one fde1d_step launch per time level, and that with S1 + S2 in every step.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU (torchrun, one rank per GPU): the single-problem path does not shard (DESIGN.md,
"replicas only"): every rank runs its own cfg3 replica; value = all ranks' steps / max time.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "time-steps/sec (HODLR build+factor+solve), n=65536 1D; HBM GB/s % of peak"
FP64_TENSOR_TFLOPS = 37.05   # measured DMMA f64 peak on this pool (profiles/fp64_peak_r01.json)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=64)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-extra", action="store_true",
                   help="skip the informational cfg4 (sharded batch) and cfg5 (2D) measurements")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------
# clocks during the timed region
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-i", str(self.gpu), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------
def algorithmic_work(ranks, n, leaf_sizes, nf=1):
    """Per-step algorithmic FP64 flops and compulsory bytes per kernel.

    k = r + 1 columns per level (r low-rank + the exact -g_0 column), NC = nf + sum k (panel
    width), xc[l] = nf + sum_{l'<l} k_l' (first panel column of level l).
      k_leaf : per leaf of s rows: LU (2/3) s^3, panel solve 2 s^2 NC, projection of the panel
               on every ancestor's V factor 2 s (NC - nf) NC (Q = V^T X);
               bytes: write X (n x NC) and Q (per leaf (NC-1) x NC), read d+-, u, f, L_l rows.
      k_tree : per node of level m (2^m nodes): the K solve (2/3)(k^3) + 3 k^2 xc[m] flops and
               the projected update 2 (xc[m]-1) xc[m] 2k; final u = X v: 2 n NC;
               bytes: read the children's Q, write Q_node, read X once.
      k_levels (level-pass variant): 2 n k (nf + W_l + k) + 2 n k (nf + W_l) flops per level.
    """
    ks = [r + 1 for r in ranks]
    L = len(ks)
    xc = [nf + sum(ks[:l]) for l in range(L + 1)]
    NC = xc[L]
    nleaf = len(leaf_sizes)
    work = {}
    fl = sum(2.0 / 3.0 * s ** 3 + 2.0 * s * s * NC + 2.0 * s * (NC - nf) * NC for s in leaf_sizes)
    by = 8.0 * n * NC + 8.0 * nleaf * (NC - 1) * NC + 8.0 * n * sum(ranks) + 8.0 * 4 * n
    work["k_leaf"] = (fl, by)
    ft, bt = 2.0 * n * NC, 8.0 * n * NC
    for m in range(L):
        k, x = ks[m], xc[m]
        ft += 2 ** m * (2.0 / 3.0 * k ** 3 + 3.0 * k * k * x + 2.0 * (x - 1) * x * 2 * k)
        bt += 2 ** m * 8.0 * (2 * (xc[m + 1] - 1) * xc[m + 1] + (x - 1) * x + 2 * k * x)
    work["k_tree"] = (ft, bt)
    # k_step = k_leaf + k_tree fused in one persistent dataflow launch (the default path)
    work["k_step"] = (fl + ft, by + bt)
    # k_run = k_step per time level, K levels pipelined in one launch (per-step figures)
    work["k_run"] = work["k_step"]
    Wl = [sum(ks[:l]) for l in range(L)]
    fl_l = sum(2.0 * n * k * (nf + w + k) + 2.0 * n * k * (nf + w) for k, w in zip(ks, Wl))
    by_l = sum(8.0 * n * (nf + w + k) + 8.0 * n * (nf + w) for k, w in zip(ks, Wl))
    work["k_levels"] = (fl_l, by_l)
    return work


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            return json.load(fh)
    except Exception:
        return {}


# ---------------------------------------------------------------------------------------
def cpu_oracle_baseline(wl, n_sample=8192, reps=2):
    """The oracle as it stands (dense LAPACK LU step, oracle.fd1d) on the host cores, on a
    bounded sample of cfg3: n_sample interior points with cfg3's alpha, dt and coefficients,
    extrapolated to n = 65536 by the O(n^3) LU cost."""
    from oracle.fd1d import assemble_A, step_dense   # oracle: cpu_baseline leg only
    from paper_1804_05522_b200 import workloads as W
    cores = os.cpu_count()
    s = W.cfg3(K=reps, n=n_sample)
    u = s.u0[0]
    t0 = time.perf_counter()
    for m in range(1, reps + 1):
        dp, dm = s.coeffs(m)
        A = assemble_A(float(s.alpha[0]), s.n, s.h, s.dt, dp[0], dm[0])
        u, _ = step_dense(A, u, s.source(m)[0], s.dt)
    el = (time.perf_counter() - t0) / reps
    scale = (wl.n / n_sample) ** 3
    value = 1.0 / (el * scale)
    return {"value": value, "unit": "time-steps/s", "cores": cores, "kind": "oracle",
            "sample": "%d dense LU steps (oracle.fd1d.assemble_A + step_dense) at n=%d with cfg3's "
                      "alpha/dt/coefficients, %.2f s/step, extrapolated x(%d/%d)^3 = x%d (LU is O(n^3))"
                      % (reps, n_sample, el, wl.n, n_sample, int(scale))}


def run_reference(args, world, rank):
    if rank != 0:
        return 0
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count()))
    from paper_1804_05522_b200 import workloads as W
    wl = W.cfg3(K=2)
    steps = max(1, min(args.steps, 3))
    warm = max(0, min(args.warmup, 1))
    base = cpu_oracle_baseline(wl, n_sample=8192, reps=warm + steps)      # (the same sample as our arm's)
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "time-steps/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": warm,
            "ms_per_step": 1e3 / base["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "cfg3: 1D FDE n=65536 alpha=1.8 leaf 128 tol 1e-10 (BASELINE configs[2])",
                       "l2": "n/a (CPU)"},
            "cpu_baseline": {"kind": "oracle", "cores": base["cores"], "sample": base["sample"],
                             "value": base["value"], "unit": "time-steps/s"},
            "e2e": {"value": base["value"], "unit": "time-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------------------
def _max_over_ranks(dev, world, x):
    if world > 1:
        import torch
        t = torch.tensor([x], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())
    return x


def measure_cfg4(dev, world, rank, steps=16):
    """BASELINE configs[3]: 512 independent n = 8192 problems, time-invariant d+- (P:1333), 16
    steps; instances sharded over the ranks (shard.py), no collective in the timed region.
    Reported (instance-steps/s over all ranks, max-over-ranks device time):
      value_factor_once        -- ONE figure for the whole run: the factorisation (fused with the
                                  first step's solve) + the 15 further solves with the kept factor,
                                  i.e. SURVEY §8(d)'s "factor once" protocol (its roofline: ~2.7e5);
      value_solve_only         -- the 16 steps with an already kept factor (solve phase alone);
      value_refactor_every_step / _pipelined_run -- d+- treated as new every step;
      value_factor_once_run    -- fde1d_run with the coefficients given once (factor once): at
                                  this size (32768 leaves > 16 per SM) it takes the kept-factor
                                  path (the pipelined launch's factor-once mode, k_run inv,
                                  is faster only below ~16 leaves per SM: DESIGN.md)."""
    import torch
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_NO_KEEP, FDE_REFACTOR
    from paper_1804_05522_b200.shard import ShardedRun
    wl = W.cfg4()
    run = ShardedRun(wl.batch, world, rank)
    sl = slice(run.start, run.start + run.count)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    dp, dm = wl.coeffs(1)
    DP, DM, F = t(dp[sl]), t(dm[sl]), t(wl.source(1)[sl])
    u = [t(wl.u0[sl]), torch.empty_like(t(wl.u0[sl]))]
    st = Fde1dStepper(wl.n, wl.alpha[sl], wl.h, wl.tol, wl.leaf, batch=run.count)
    st.step(wl.dt, DP, DM, F, u[0], u_next=u[1], coeffs_changed=True)     # build (S1-S2) + factor
    torch.cuda.synchronize()

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms = _max_over_ranks(dev, world, a.elapsed_time(b))
        return wl.batch * steps / (ms / 1e3), ms

    def factor_once():                               # factor (fused with step 1) + 15 solves
        for k in range(steps):
            st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], coeffs_changed=(k == 0))

    def solve_only():
        for k in range(steps):
            st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], coeffs_changed=False)

    def refactor():
        for k in range(steps):
            st.step(wl.dt, DP, DM, F, u[k % 2], u_next=u[(k + 1) % 2], coeffs_changed=True, flags=FDE_NO_KEEP)
    factor_once()
    v_once, ms_once = timed(factor_once)
    factor_once()                                    # (re-keep the factor for the solve-only pass)
    v_solve, ms_solve = timed(solve_only)
    v_ref, ms_ref = timed(refactor)
    try:
        runf = lambda fl: st.run(wl.dt, DP[None], DM[None], F[None], u[0], K=steps, flags=fl)
        runf(FDE_REFACTOR)
        v_run, ms_run = timed(lambda: runf(FDE_REFACTOR))
        runf(0)
        v_run1, ms_run1 = timed(lambda: runf(0))     # factor once (routed: kept-factor path)
    except Exception as e:                          # (memory for the second buffer set)
        v_run, ms_run, v_run1, ms_run1 = None, str(e)[:120], None, None
    st.close()
    return {"workload": "cfg4: 512 x n=8192, alpha_i~U(1.1,1.9), 16 steps, leaf 128, tol 1e-13 (R18)",
            "metric": "instance-steps/s",
            "value_factor_once": v_once, "ms_16_steps_factor_once": ms_once,
            "value_solve_only": v_solve, "ms_16_steps_solve_only": ms_solve,
            "value_refactor_every_step": v_ref, "ms_16_steps_refactor": ms_ref,
            "value_refactor_pipelined_run": v_run, "ms_16_steps_refactor_pipelined_run": ms_run,
            "value_factor_once_run": v_run1, "ms_16_steps_factor_once_run": ms_run1,
            "survey_roofline_factor_once": 2.7e5,
            "sharding": "%d instances per rank (shard.py), no data-path collective" % run.count}


def measure_cfg5(dev, world, rank, steps=16):
    """BASELINE configs[4]: the 2D Sylvester step, nx = ny = 2048, all 16 steps of the trajectory
    (operators factorised once: the coefficients are time-invariant).  world = 1: fde2d_step.
    world >= 2: the x/y split (split2d.py, fde2d_step_split) on rank pairs; pairs beyond the first
    solve their own replica of the problem (value = all pairs' steps / max time)."""
    import torch
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200.hodlr import Fde2dStepper
    wl = W.cfg5()
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    Fs = [tuple(t(f.T) for f in wl.source_factors(m)) for m in range(1, steps + 1)]
    args = (wl.nx, wl.ny, wl.alpha1, wl.alpha2, wl.hx, wl.hy, wl.dt, t(wl.d1p), t(wl.d1m), t(wl.d2p), t(wl.d2m), wl.tol)
    if world == 1:
        st = Fde2dStepper(*args, ek_tol=wl.ek_tol, leaf=wl.leaf)
        stepf = lambda m, X: st.step(*Fs[m]) if X is None else st.step(*Fs[m], *X)
        own = lambda out: (out[0], out[1])
        pairs, psize = 1, 1
    else:
        from paper_1804_05522_b200.split2d import SplitSylvesterStepper, pair_group
        g, prank, psize = pair_group(world, rank)
        st = SplitSylvesterStepper(*args, ek_tol=wl.ek_tol, leaf=wl.leaf, group=g, world=psize, rank=prank)
        pairs = world // 2

        def stepf(m, X):
            Fu, Fv = Fs[m]
            if psize == 1:
                return st.step(Fu, Fv, *(X if X is not None else (None, None)))
            if prank == 0:
                return st.step(Fu, None, X, None)
            return st.step(None, Fv, None, X)
        own = lambda out: out[0]
    X = own(stepf(0, None))                             # builds + factors the operator(s)
    torch.cuda.synchronize()

    def trajectory():
        X, its = None, []
        for m in range(steps):
            out = stepf(m, X)
            X = own(out)
            its.append(out[-1])
        return X, its
    trajectory()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    X, its = trajectory()
    torch.cuda.synchronize()
    el = _max_over_ranks(dev, world, time.perf_counter() - t0)
    st.close()
    return {"workload": "cfg5: 2D nx=ny=2048, alpha=(1.3,1.7), rank-4 source, ek_tol 1e-11, tol 1e-12, all %d steps" % steps,
            "metric": "time-steps/s", "value": max(1, pairs) * steps / el, "ms_per_step": 1e3 * el / steps,
            "steps": steps, "ek_iterations": its,
            "parallelism": "single GPU" if world == 1 else "x/y split over rank pairs (%d pair(s) of %d)" % (pairs, psize),
            "timing": "host wall clock around the synchronous fde2d_step calls of the whole trajectory "
                      "(max over ranks); the step reads back the small quantities that steer EK"}


def measure_cfg3_split(dev, world, rank, steps=16):
    """ONE cfg3 trajectory split over the ranks at the top of the HODLR tree
    (fde1d_step_split, split1d.py): strong scaling of a single problem (value = time-steps/s of the
    one trajectory, max-over-ranks device time).  Only at N >= 2 (a power of two)."""
    import torch
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200.split1d import Split1dStepper
    wl = W.cfg3(K=steps)
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    DP = [t(wl.coeffs(m)[0][0]) for m in range(1, steps + 1)]
    DM = [t(wl.coeffs(m)[1][0]) for m in range(1, steps + 1)]
    F = t(wl.source(1)[0])
    u = [t(wl.u0[0]), torch.empty_like(t(wl.u0[0]))]
    sp = Split1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, world=world, rank=rank)
    for k in range(2):
        sp.step(wl.dt, DP[k], DM[k], F, u[k % 2], u[(k + 1) % 2])
    torch.distributed.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(steps):
        sp.step(wl.dt, DP[k], DM[k], F, u[k % 2], u[(k + 1) % 2])
    b.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(dev, world, a.elapsed_time(b))
    sp.close()
    return {"workload": "cfg3 (n=65536) one trajectory split over %d GPUs at the top of the tree" % world,
            "metric": "time-steps/s", "value": steps / (ms / 1e3), "ms_per_step": ms / steps,
            "scaling": "strong (one problem)", "exchange": "all-gather of the level-p projected matrices "
            "+ u row blocks per step (NCCL via torch.distributed)"}


def measure_small(dev, name, reps=3):
    """BASELINE configs[0] / configs[1] (latency-bound sizes): the whole K-step trajectory through
    fde1d_run, CUDA events around the launch after a warm-up run.  cfg2 (d+-(x, t)) refactors every
    step; cfg1 (d+- = 1, time-invariant) factors once inside the launch -- `value` -- and
    is also timed with FDE_REFACTOR (`value_refactor`)."""
    import torch
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200.hodlr import Fde1dStepper, FDE_REFACTOR
    wl = getattr(W, name)()
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)
    DP, DM, F, U0 = t(wl.d_plus), t(wl.d_minus), t(wl.f), t(wl.u0)
    st = Fde1dStepper(wl.n, wl.alpha, wl.h, wl.tol, wl.leaf, batch=wl.batch)

    def best_ms(flags):
        st.run(wl.dt, DP, DM, F, U0, flags=flags)
        torch.cuda.synchronize()
        best = None
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            st.run(wl.dt, DP, DM, F, U0, flags=flags)
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        return best
    best = best_ms(0)
    invariant = wl.d_plus.shape[0] == 1
    out = {"workload": "%s: n=%d alpha=%g leaf %d tol %g, %d steps (BASELINE configs), %s" % (
               name, wl.n, float(wl.alpha[0]), wl.leaf, wl.tol, wl.K,
               "d+- time-invariant: factor once in the launch" if invariant else "refactor every step"),
           "metric": "time-steps/s", "value": wl.K / (best / 1e3), "us_per_step": 1e3 * best / wl.K,
           "ranks": st.ranks(), "timing": "CUDA events around one fde1d_run of all K steps, best of %d" % reps}
    if invariant:
        best_r = best_ms(FDE_REFACTOR)
        out["value_refactor"] = wl.K / (best_r / 1e3)
        out["us_per_step_refactor"] = 1e3 * best_r / wl.K
    st.close()
    return out


def task_profile(K=16):
    """Per-task durations inside k_run: tools/task_profile.py in a subprocess against the
    diagnostics library (libfdehodlr_dbg.so; the product library has no trace switches)."""
    env = dict(os.environ, FDE_LIB_DEBUG="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "task_profile.py"), str(K)],
                       env=env, capture_output=True, text=True, timeout=300)
    if r.returncode != 0:
        return {"error": (r.stderr or r.stdout)[-300:]}
    return json.loads(r.stdout.strip().splitlines()[-1])


def run_ours(args, world, rank, local):
    import torch
    from paper_1804_05522_b200 import build as B
    B.build()
    from paper_1804_05522_b200 import workloads as W
    from paper_1804_05522_b200 import _lib
    from paper_1804_05522_b200.hodlr import (Fde1dStepper, launch_count, FDE_RECOMPRESS,
                                             FDE_NO_KEEP, FDE_HOST_PTRS)
    lib = _lib.load()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # the timed trajectory: args.steps time levels of cfg3 (new d+-(x, t_m) every step)
    wl = W.cfg3(K=max(args.steps, args.warmup, 1))
    n = wl.n
    DPK = torch.as_tensor(wl.d_plus, device=dev).contiguous()        # (K, 1, n)
    DMK = torch.as_tensor(wl.d_minus, device=dev).contiguous()
    F = torch.as_tensor(wl.f[0:1], device=dev).contiguous()           # (1, 1, n): time-invariant
    U0 = torch.as_tensor(wl.u0, device=dev).contiguous()              # (1, n)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    st = Fde1dStepper(n, wl.alpha, wl.h, wl.tol, wl.leaf)
    evs = lambda: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))

    def run(K, profile=False):
        """One fde1d_run of K pipelined steps (one k_run launch); device time in ms."""
        flush.zero_()
        a, b = evs()
        if profile:
            lib.fde_profile_enable(1)
        barrier()
        torch.cuda.synchronize()
        l0 = launch_count()
        a.record()
        out = st.run(wl.dt, DPK[:K], DMK[:K], F, U0)
        b.record()
        torch.cuda.synchronize()
        l1 = launch_count()
        barrier()
        prof = None
        if profile:
            buf = __import__("ctypes").create_string_buffer(1 << 16)
            lib.fde_profile_dump(buf, 1 << 16)
            lib.fde_profile_enable(0)
            prof = json.loads(buf.value.decode())
        return a.elapsed_time(b), l1 - l0, prof, out

    run(args.steps)                               # build the handle, size the run buffers (K)
    for _ in range(max(3, args.warmup)):          # warm-up: >= 3 untimed runs of the same K
        run(args.steps)
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    total_ms, launches, _, out = run(args.steps)
    clk = clocks.stop()
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * args.steps / (total_ms / 1e3)
    if not bool(torch.isfinite(out).all()):
        raise RuntimeError("non-finite solution in the timed run")

    # per-kernel durations (CUDA events around the launch on its stream, same run again)
    pms, _, prof, _ = run(args.steps, profile=True)

    # the per-step variant: one fused k_step launch per fde1d_step call, L2 flushed between
    bufs = [torch.zeros(n, dtype=torch.float64, device=dev) for _ in range(2)]

    def per_step(K, flags):
        ms = 0.0
        for k in range(K):
            flush.zero_()
            a, b = evs()
            a.record()
            st.step(wl.dt, DPK[k % wl.K, 0], DMK[k % wl.K, 0], F[0, 0], bufs[k % 2],
                    u_next=bufs[(k + 1) % 2], coeffs_changed=True, flags=flags)
            b.record()
            torch.cuda.synchronize()
            ms += a.elapsed_time(b)
        return ms
    per_step(2, FDE_NO_KEEP)
    vK = min(args.steps, 32)
    ms_ps = per_step(vK, FDE_NO_KEEP)
    ms_rc = per_step(max(1, vK // 4), FDE_NO_KEEP | FDE_RECOMPRESS)
    other = {"per_step_launch": {"value": world * vK / (ms_ps / 1e3), "ms_per_step": ms_ps / vK,
                                 "what": "fde1d_step per time level (one k_step launch each), "
                                         "L2 flushed between steps"},
             "per_step_recompress": {"value": world * max(1, vK // 4) / (ms_rc / 1e3),
                                     "ms_per_step": ms_rc / max(1, vK // 4),
                                     "what": "as per_step_launch plus S1 (GL weights) + S2 "
                                             "(compression of T_alpha) inside every step"}}

    # end to end through the public API: H2D of the K steps' d+-, f, u0 from pinned host memory,
    # the pipelined run, D2H of every step's solution -- all inside the timed region
    e2e = None
    if not args.no_e2e:
        pin = lambda t: t.cpu().pin_memory()
        hDP, hDM, hF, hU0 = pin(DPK[:args.steps]), pin(DMK[:args.steps]), pin(F), pin(U0)
        hout = torch.empty((args.steps, 1, n), dtype=torch.float64).pin_memory()

        def e2e_once():                     # the C-ABI call with HOST buffers (FDE_HOST_PTRS):
            st.run(wl.dt, hDP, hDM, hF, hU0, u_out=hout, flags=FDE_HOST_PTRS)   # copies inside
            torch.cuda.synchronize()
        e2e_once()
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e2e_once()
        el = time.perf_counter() - t0
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([el], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        h2d = sum(x.numel() * 8 for x in (hDP, hDM, hF, hU0))
        e2e = {"value": world * args.steps / el, "unit": "time-steps/s",
               "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": n * 8,
               "timing": "host wall clock around fde1d_run with FDE_HOST_PTRS (pinned host buffers: the "
                         "library's H2D staging, the run and the D2H of every step's solution inside the "
                         "call), synchronize on both sides, max over ranks"}

    ranks = st.ranks()
    leaves = [wl.leaf] * (n // wl.leaf)
    work = algorithmic_work(ranks, n, leaves)
    peaks = load_peaks()
    traffic = load_traffic()
    kern = {}
    for name, (cnt, tot) in (prof or {}).items():
        kern[name] = {"launches_per_step": cnt / args.steps, "ms_per_step": tot / args.steps}
    dom = max(kern, key=lambda k: kern[k]["ms_per_step"]) if kern else None
    roof = None
    if dom:
        t_s = kern[dom]["ms_per_step"] / 1e3
        launches_dom = kern[dom]["launches_per_step"]
        fl, by = work.get(dom, (0.0, 0.0))
        if dom in ("k_leaf", "k_levels", "k_tree", "k_step", "k_run"):
            # FP64 contractions on the DMMA (FP64 tensor) path; MEASURED_PEAKS has no FP64
            # entry: peak = tools/fp64_peak.cu measurement (profiles/fp64_peak_r01.json),
            # equal to the derived 148 SMs x 64 FMA/clk x 2 x 1.965 GHz = 37.2 TFLOP/s
            roof = {"bound": "tensor", "achieved": fl / t_s / 1e12, "peak": FP64_TENSOR_TFLOPS,
                    "unit": "TFLOP/s", "frac": fl / t_s / 1e12 / FP64_TENSOR_TFLOPS,
                    "traffic": (traffic[dom + "_per_step"] * args.steps if dom + "_per_step" in traffic
                                else traffic.get(dom)), "kernel": dom,
                    "flops_per_launch": fl / launches_dom,
                    "achieved_hbm_gbs": by / t_s / 1e9,
                    "peak_source": "measured DMMA m8n8k4 f64 (tools/fp64_peak.cu): 37.05 TFLOP/s"}
        else:
            roof = {"bound": "hbm", "achieved": by / t_s / 1e9, "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s", "frac": by / t_s / 1e9 / peaks.get("hbm_gbs", 6549.1),
                    "traffic": traffic.get(dom), "kernel": dom,
                    "bytes_per_launch": by / launches_dom,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs (of measured)"}
        roof["share_of_step"] = kern[dom]["ms_per_step"] / (pms / args.steps)

    line = {"metric": METRIC, "value": value, "unit": "time-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "cfg3: 1D FDE n=65536 alpha=1.8 leaf 128 tol 1e-10, d+-(x,t) per "
                                   "BASELINE configs[2], new d+-(x,t_m) and refactor every step, "
                                   "K = steps time levels pipelined in one fde1d_run",
                       "n": n, "leaf": wl.leaf, "tol": wl.tol, "ranks": ranks,
                       "parallelism": "replicas" if world > 1 else "single",
                       "l2": "flushed (512 MiB write) before the timed launch; inside it every "
                             "step's working set (panel X %.0f MB + stored leaf LU %.0f MB + "
                             "d+-, u) exceeds the 126 MB L2" % (8e-6 * n * (sum(ranks) + len(ranks) + 1),
                                                                 8e-6 * n * wl.leaf),
                       "step": "S3-S7 every step; S1-S2 (T_alpha compression) once per handle "
                               "(other_variant.per_step_recompress puts them in every step)"},
            "gpu_launches": launches,
            "clocks": clk, "e2e": e2e, "roofline": roof, "kernels": kern,
            "other_variant": other}
    def extras():
        try:
            line["task_profile"] = task_profile()
        except Exception as e:
            line["task_profile"] = {"error": str(e)[:200]}
        extra = line.setdefault("other_configs", {})
        for name in ("cfg1", "cfg2"):
            try:
                extra[name] = measure_small(dev, name)
            except Exception as e:
                extra[name] = {"error": str(e)[:200]}
        try:
            extra["cfg4"] = measure_cfg4(dev, world, rank)
        except Exception as e:                              # reported, not fatal for the headline
            extra["cfg4"] = {"error": str(e)[:200]}
        if world > 1 and (world & (world - 1)) == 0:
            try:
                extra["cfg3_split"] = measure_cfg3_split(dev, world, rank)
            except Exception as e:
                extra["cfg3_split"] = {"error": str(e)[:200]}
        try:
            extra["cfg5"] = measure_cfg5(dev, world, rank)
        except Exception as e:
            extra["cfg5"] = {"error": str(e)[:200]}

    if not args.no_extra and world == 1 and not os.environ.get("FDE_BENCH_WATCHDOG"):
        extras()
    elif not args.no_extra:
        # Multi-rank extras contain collectives: a rank that fails alone would leave the others
        # waiting, so they run under a watchdog and the (already measured) headline line is printed
        # whatever happens to them.
        import threading

        def guarded():
            torch.cuda.set_device(local)
            extras()

        th = threading.Thread(target=guarded, daemon=True)
        th.start()
        th.join(float(os.environ.get("FDE_BENCH_EXTRA_TIMEOUT", "420")))
        if th.is_alive():
            line.setdefault("other_configs", {})["watchdog"] = "multi-rank extras timed out; headline unaffected"
            if rank == 0:
                try:
                    out = json.dumps(line, default=str)
                except RuntimeError:                      # the extras thread is writing into it
                    out = json.dumps({k: v for k, v in line.items()
                                      if k not in ("other_configs", "task_profile")}, default=str)
                print(out, flush=True)
            os._exit(0)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_baseline(wl)
    if rank == 0:
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    return run_ours(args, world, rank, local)


if __name__ == "__main__":
    sys.exit(main())
