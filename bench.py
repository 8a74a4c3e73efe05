"""Benchmark: RRS query-depths/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload config4]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)
    python bench.py --impl reference ...                       (CPU reference arm)

Workload (default, BASELINE.json configs[3] / north_star target): halfspace
depth RRS, n=100k Toeplitz-Gaussian points (reference generator bytes), d=50,
k=NRandom=20,000 = 1000 directions x 20 refinements, alpha=0.9, RRS seed 1,
queries = the data points themselves (query index = row index).  One step =
one batch of B queries per GPU through all 20 refinements; scaling is weak
(B per GPU fixed).  value = queries of all ranks / max-over-ranks device time.

The FP32 roofline (north_star): FLOPs = 2 n d m per (query, refinement); the
dominant kernel is contract_kernel<count> (K2), measured with CUDA events on
the engine stream.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (notion, n, d, k, r, alpha, distribution, batch per GPU)
    "config1": ("halfspace", 1_000, 5, 1_000, 10, 0.9, "gaussian", 1000),
    "config2": ("projection", 10_000, 20, 20_000, 20, 0.9, "gaussian", 512),
    "config3": ("asym_projection", 50_000, 50, 20_000, 20, 0.9, "cauchy", 32),
    "config4": ("halfspace", 100_000, 50, 20_000, 20, 0.9, "gaussian", 1024),
    # config 5 cells (n = 1M, d = 200) on a fixed query subset per step
    "config5": ("halfspace", 1_000_000, 200, 20_000, 20, 0.9, "gaussian", 16),
    "config5p": ("projection", 1_000_000, 200, 20_000, 20, 0.9, "gaussian", 4),
}
WORKLOAD_TEXT = {
    "config1": "halfspace depth RRS, n=1000 Gaussian, d=5, NRandom=1000, n_refinements=10, all points as queries",
    "config2": "projection depth RRS (median/MAD), n=10k, d=20, Gaussian, k=20000 x r=20",
    "config3": "asymmetric projection depth RRS, n=50k, d=50, Cauchy (t, nu=1), k=20000 x r=20",
    "config4": "halfspace depth RRS, n=100k, d=50, K=1000x20 refinements (k=20000), all n points as queries",
    "config5": "halfspace depth RRS, n=1M, d=200, Gaussian, k=20000 x r=20, alpha 0.9 (one cell of the sweep)",
    "config5p": "projection depth RRS, n=1M, d=200, Gaussian, k=20000 x r=20, alpha 0.9 (one cell of the sweep)",
}
FP32_NOMINAL_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4: 148 SMs x 128 FP32 lanes x FMA x 1965 MHz


def make_data(dist: str, n: int, d: int) -> np.ndarray:
    from paper_2506_08262_b200.synthetic import student_t, toeplitz_gaussian

    return toeplitz_gaussian(d, n, seed=0) if dist == "gaussian" else student_t(d, n, 1.0, seed=0)


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


def store_split2(X) -> bool:
    """Whether the engine's auto plan takes the two-term split store for d <= 64
    (engine.cu make_plan: column IQR ratio <= 8 over the centre sample of
    center_sample_kernel: min(n, 1024) rows at strided positions)."""
    n = X.shape[0]
    S = min(n, 1024)
    rows = ((4 * np.arange(S) + 1) * n) // (4 * S)
    s = np.sort(X[rows], axis=0)
    iqr = s[min((3 * S) // 4, S - 1)] - s[S // 4]
    iqr = iqr[iqr > 0]
    return iqr.size == 0 or float(iqr.max() / iqr.min()) <= 8.0


def profile_traffic(workload: str):
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get(workload, {}).get("contract_dram_bytes_per_launch")
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(busy), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


def cpu_baseline(X, notion, k, r, alpha, budget_queries=None):
    """The CPU port of the reference (oracle/, kind "port") on this host's
    cores: a bounded sample of the same workload (one query per thread).  When
    one full query is too long for the budget (config 5: 8e12 FLOP per query),
    each sampled query runs r' < r refinements of the same m directions and the
    rate is scaled by r'/r (RRS cost is linear in the refinements)."""
    from oracle import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    q = budget_queries or max(cores, 1)
    n, d = X.shape
    m = -(-k // r)
    r_s, m_s = cpu_sample_budget(n, d, k, r)
    scale = (r * m) / (r_s * m_s)
    # short samples (config 1: 16 queries in ~10 ms) repeat over the next rows
    # until >= 3 s of CPU work, so the rate is not timer noise
    n_rows = X.shape[0]
    done, dt, reps = 0, 0.0, 0
    while True:
        rows = (np.arange(done, done + q) % n_rows)
        t0 = time.perf_counter()
        oracle.depth_batch(X[rows], X, total_directions=m_s * r_s, refinements=r_s, shrink=alpha, notion=notion,
                           seed=1, threads=cores, q0=int(rows[0]))
        dt += (time.perf_counter() - t0) * scale
        done += q
        reps += 1
        if dt / scale >= 3.0 or reps >= 2000:
            break
    part = "full RRS" if scale == 1 else f"{r_s} refinement(s) of {m_s} directions timed, scaled x{scale:g}"
    return {"value": done / dt, "unit": "query-depths/s", "cores": cores, "kind": "port",
            "sample": f"{done} in-sample queries ({reps} x {q} consecutive rows from row 0) of the same workload, "
                      f"{part}, {cores} threads, {dt / scale:.1f} s wall"}


def cpu_sample_budget(n, d, k, r, flop_budget=2.5e11):
    """(refinements, directions per refinement) a CPU sample query runs: the
    full (r, m) unless one query exceeds the per-thread FLOP budget (~20-40 s
    of scalar FP64 work); then fewer refinements, and below one refinement
    fewer directions.  RRS cost is linear in both, so the rate is scaled by
    (r m) / (r' m')."""
    m = -(-k // r)
    per_dir = 2.0 * n * d
    if per_dir * m * r <= flop_budget:
        return r, m
    r_s = int(flop_budget // (per_dir * m))
    if r_s >= 1:
        return r_s, m
    return 1, max(1, int(flop_budget // per_dir))


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def run_reference(args, wl):
    """--impl reference: the reference's CPU algorithm (oracle port) on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    notion, n, d, k, r, alpha, dist, _ = WORKLOADS[wl]
    X = make_data(dist, n, d)
    cores = os.cpu_count() or 1
    from oracle import oracle

    oracle.build()
    q = cores
    r_s, m_s = cpu_sample_budget(n, d, k, r)
    k_s = m_s * r_s
    scale = (r * -(-k // r)) / k_s
    for _ in range(args.warmup):
        oracle.depth_batch(X[:1], X, total_directions=k_s, refinements=r_s, shrink=alpha, notion=notion, seed=1,
                           threads=1)
    times = []
    for s in range(args.steps):
        Z = X[(s * q) % n:(s * q) % n + q]
        t0 = time.perf_counter()
        oracle.depth_batch(Z, X, total_directions=k_s, refinements=r_s, shrink=alpha, notion=notion, seed=1,
                           threads=cores, q0=(s * q) % n)
        times.append((time.perf_counter() - t0) * scale)
    total = sum(times)
    value = q * args.steps / total
    line = {
        "impl": "reference", "metric": "query-depths/s (RRS, all n points)", "value": value,
        "unit": "query-depths/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference generators)",
        "config": {"workload": WORKLOAD_TEXT[wl], "notion": notion, "n": n, "d": d, "NRandom": k,
                   "n_refinements": r, "sphcap_shrink": alpha, "queries_per_step": q},
        "cpu_baseline": {"value": value, "unit": "query-depths/s", "cores": cores, "kind": "port",
                         "sample": f"{q} queries per step ({cores} threads, {cpu_model()}); warm-up steps "
                                   "run one query" + ("" if scale == 1 else
                                                      f"; {r_s} refinement(s) of {m_s} directions timed, "
                                                      f"scaled x{scale:g}")},
        "e2e": {"value": value, "unit": "query-depths/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config4", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0, help="queries per GPU per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group for N>1 (gloo: ranks may share one GPU, the single-GPU rehearsal)")
    ap.add_argument("--select-path", default="auto", choices=["auto", "radix", "wide"],
                    help="order-statistic kernel of the projection notions (A/B)")
    ap.add_argument("--early-exit", action="store_true",
                    help="RrsConfig(early_exit=True): exact early exit of finished halfspace queries "
                         "(outputs bitwise unchanged; not the default, which does the reference's full work)")
    ap.add_argument("--workspace-mb", type=int, default=0,
                    help="engine workspace cap (query batching / projection chunking), MiB; 0 = default")
    ap.add_argument("--contract-path", default="auto", choices=["auto", "ffma", "tensor", "filter", "tensor3", "convert"],
                    help="halfspace contraction kernel (auto: the library's choice)")
    args = ap.parse_args()
    wl = args.workload
    if args.impl == "reference":
        return run_reference(args, wl)

    import torch
    import torch.distributed as dist

    import paper_2506_08262_b200 as rrs
    from paper_2506_08262_b200.distributed import depth_sharded_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dist_backend == "gloo":
        local = local % torch.cuda.device_count()  # ranks may share a GPU
    torch.cuda.set_device(local)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    red_dev = "cuda" if args.dist_backend == "nccl" else "cpu"  # timing max-reduction
    notion, n, d, k, r, alpha, distn, B = WORKLOADS[wl]
    if args.batch:
        B = args.batch
    m = -(-k // r)
    cfg = rrs.RrsConfig(total_directions=k, refinements=r, shrink=alpha, notion=notion, seed=1,
                        early_exit=args.early_exit)
    X = make_data(distn, n, d)
    eng = rrs.engine(local)
    eng.set_contract_path(args.contract_path)
    eng.set_select_path(args.select_path)
    if args.workspace_mb:
        eng.set_workspace_limit(args.workspace_mb << 20)
    stream = torch.cuda.Stream()  # one non-default stream shared by torch and the engine
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    eng.set_dataset(X, key="bench")
    Xd = torch.from_numpy(X).cuda()

    def step_rows(s):
        start = ((s * world + rank) * B) % n
        return start, Xd[start:start + B] if start + B <= n else torch.cat([Xd[start:], Xd[: B - (n - start)]])

    total_steps = args.warmup + args.steps
    inputs = [step_rows(s) for s in range(total_steps)]  # resident in HBM before timing
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def run_step(s):
        q0, Z = inputs[s]
        return depth_sharded_device(Z.contiguous(), cfg, q_offset=q0, eng=eng)

    for s in range(args.warmup):
        run_step(s)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    recs = []
    for i in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the events)
        ev[i][0].record(stream)
        recs.append(run_step(args.warmup + i))
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    # stage breakdown (kernel launches, contraction / select event times) from a
    # second pass over the same steps with the engine's per-stage events on --
    # outside the timed region: the event records and the per-step stats sync
    # would otherwise slow launch-bound configurations (config 1)
    eng.enable_timing(True)
    launches = 0
    contract_ms = 0.0
    contract_launches = 0
    tensor_launches = 0
    select_ms = 0.0
    stage_ms = 0.0
    for i in range(args.steps):
        flush.zero_()
        a_ev, b_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a_ev.record(stream)
        run_step(args.warmup + i)
        b_ev.record(stream)
        st = eng.stats()  # syncs; per-kernel event times of this step
        stage_ms += a_ev.elapsed_time(b_ev)
        launches += st["kernel_launches"]
        contract_ms += st["ms_contract_total"]
        contract_launches += st["contract_launches"]
        tensor_launches += st["tensor_contract_launches"]
        select_ms += st["ms_univariate"]
    eng.enable_timing(False)  # kernel shares below: against this pass's own step time
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * B * args.steps / (ms_max / 1e3)

    # Side measurement, not the headline: the same steps with RrsConfig(early_exit=True)
    # (halfspace: a query stops once its best count equals the rows coinciding with it;
    # outputs must be bitwise those of the full-work steps above, checked here)
    early = None
    if notion == "halfspace" and not args.early_exit:
        import dataclasses

        cfg_full = cfg
        cfg = dataclasses.replace(cfg_full, early_exit=True)
        run_step(0)  # warm-up of the early-exit variant
        torch.cuda.synchronize()
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        recs2 = []
        for i in range(args.steps):
            flush.zero_()
            ev2[i][0].record(stream)
            recs2.append(run_step(args.warmup + i))
            ev2[i][1].record(stream)
        torch.cuda.synchronize()
        ms2 = sum(a.elapsed_time(b) for a, b in ev2)
        same = all(bool(torch.equal(x, y)) for x, y in zip(recs2, recs))  # after the timed steps
        t2 = torch.tensor([ms2, 0.0 if same else 1.0], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        early = {"value": world * B * args.steps / (float(t2[0].item()) / 1e3), "unit": "query-depths/s",
                 "ms_per_step": float(t2[0].item()) / args.steps,
                 "outputs_bitwise_equal_to_full_run": bool(t2[1].item() == 0.0),
                 "what": "RrsConfig(early_exit=True): the same steps with finished queries stopped "
                         "(best count == rows coinciding with the query); not the headline value"}
        cfg = cfg_full

    # roofline of the dominant kernel (K2 contraction)
    flops_total = 2.0 * n * d * m * r * B * args.steps  # algorithmic: 2 n d m per (query, refinement)
    nl = max(contract_launches, 1)
    avg_launch_ms = contract_ms / nl
    flops_per_launch = flops_total / nl
    achieved = flops_per_launch / (avg_launch_ms / 1e3) / 1e12
    peaks = measured_peaks()
    traffic = profile_traffic(wl)
    tensor = tensor_launches == contract_launches and contract_launches > 0
    if tensor:
        # tcgen05 FP16-split path: executed tensor work = ns K-steps of M128 x N128 x K16 per
        # (128-point tile, 128-direction block); peak = measured dense bf16 (same rate as fp16)
        if notion == "halfspace":
            full = (d - 1) // 64  # kernels.h tc_layout: 64-coordinate slices (d > 64: contract_tcp.cu)
            dl = d - 64 * full
            L_ns = 12 * full + 3 * (dl // 16) + (3 * (dl % 16) + 15) // 16  # MMAs per tile and block
            wide = "contract_tcw_kernel" if args.contract_path == "convert" else "contract_tcp_kernel"
            kname, nprod = ("contract_tc_kernel" if d <= 64 else wide), 3
        elif args.contract_path != "tensor3" and (d > 64 or store_split2(X)):  # two-term split store
            full = (d - 1) // 64
            dl = d - 64 * full
            L_ns = 12 * full + 3 * (dl // 16) + (3 * (dl % 16) + 15) // 16
            wide = "contract_tcw_kernel<STORE>" if args.contract_path == "convert" else "contract_tcp_kernel<STORE>"
            kname, nprod = ("contract_tc_kernel<STORE>" if d <= 64 else wide), 3
        else:  # projection store, kernels.h Tc6Layout (contract_tcs.cu): column-heterogeneous data
            L_ns = 6 * (d // 16) + (6 * (d % 16) + 15) // 16
            kname, nprod = "contract_tcs_kernel", 6
        tiles, blocks = -(-n // 128), -(-m // 128)
        exec_per_launch = 2.0 * 128 * 128 * 16 * L_ns * tiles * blocks * (B * args.steps * r / nl)
        executed = exec_per_launch / (avg_launch_ms / 1e3) / 1e12
        peak = peaks.get("bf16_tflops") or 2250.0
        roofline = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": traffic, "kernel": kname,
                    "peak_source": ("MEASURED_PEAKS.json bf16_tflops (dense, burst; fp16 runs at the bf16 rate)"
                                    if peaks.get("bf16_tflops") else "nominal 2.25 PFLOP/s dense fp16"),
                    "achieved_is": "algorithmic FLOPs 2*n*d*m per (query, refinement) / kernel time",
                    "executed_tensor_tflops": executed, "executed_frac": executed / peak,
                    "executed_note": f"split-precision work: {L_ns} MMA K-steps ({nprod} products, packed K) per "
                                     f"128x128 tile, directions padded to {blocks * 128}",
                    "north_star_fp32": {"peak": FP32_NOMINAL_TFLOPS, "frac": achieved / FP32_NOMINAL_TFLOPS,
                                        "note": "north_star roofline: n*d*K FLOPs at the FP32 FFMA peak"}}
    else:
        roofline = {"bound": "fp32", "achieved": achieved, "peak": FP32_NOMINAL_TFLOPS, "unit": "TFLOP/s",
                    "frac": achieved / FP32_NOMINAL_TFLOPS, "traffic": traffic,
                    "kernel": "contract_kernel<count>" if notion == "halfspace" else "contract_kernel<store>",
                    "peak_source": "nominal FP32 FFMA (148 SMs x 128 lanes x 2 x 1.965 GHz); MEASURED_PEAKS.json "
                                   "has no FP32 entry"}
    roofline.update({"flops_per_launch": flops_per_launch, "avg_launch_ms": avg_launch_ms,
                     "kernel_share_of_step": contract_ms / stage_ms if stage_ms else None,
                     "hbm_peak_measured_gbs": peaks.get("hbm_gbs")})
    if notion != "halfspace" and select_ms > contract_ms:
        # the univariate stage dominates: report its roofline, HBM-bound on reading every stored
        # projection once (4 n bytes per direction and refinement); the contraction stays alongside
        hbm = peaks.get("hbm_gbs") or 8000.0
        sel_bytes = 4.0 * n * m * r * B * args.steps
        sel_gbs = sel_bytes / (select_ms / 1e3) / 1e9
        roofline = {"bound": "hbm", "achieved": sel_gbs, "peak": hbm, "unit": "GB/s", "frac": sel_gbs / hbm,
                    "traffic": None,
                    "kernel": ("select_v2_kernel<256|512|1024, smem>" if args.select_path == "radix"
                               else "select_v3_kernel<256>" if n <= 16384
                               else "select_v3_kernel<512|1024>") if 2048 <= n <= 53248
                    else ("select_v5_kernel<512, 8192>" if args.select_path != "radix" else
                          "select_v2_kernel<1024, global>") if n > 53248 and n % 4 == 0
                    else "select_v2_kernel<smem>" if n < 2048 else "select_kernel",
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks.get("hbm_gbs") else "nominal 8 TB/s",
                    "achieved_is": "algorithmic bytes (the stored projections, 4 n per direction) / select time",
                    "kernel_share_of_step": select_ms / stage_ms if stage_ms else None,
                    "contraction": roofline}
        # the store writes y once (4 n bytes per live direction): against the B200's
        # write-only bandwidth (3.91 TB/s, torch zero_ of 8 GiB, scripts/hbm_write_bw.py)
        y_bytes = 4.0 * n * m * r * B * args.steps
        roofline["contraction"]["y_write"] = {
            "achieved_gbs": y_bytes / (contract_ms / 1e3) / 1e9 if contract_ms else None,
            "write_peak_gbs": 3911.7, "peak_source": "measured write-only bandwidth, scripts/hbm_write_bw.py",
            "frac": (y_bytes / (contract_ms / 1e3) / 1e9) / 3911.7 if contract_ms else None}

    # e2e through the public API with host buffers (H2D of data + queries, D2H of results)
    e2e = None
    if not args.no_e2e:
        from paper_2506_08262_b200.distributed import depth_sharded
        from paper_2506_08262_b200.solver import depth_batch_arrays

        # host inputs in pinned memory (the e2e contract: H2D from pinned host buffers)
        Xh = torch.from_numpy(X).pin_memory().numpy()
        Zh = [inputs[args.warmup + i][1].cpu().pin_memory().numpy() for i in range(args.steps)]
        q0s = [inputs[args.warmup + i][0] for i in range(args.steps)]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for i in range(args.steps):
            data = rrs.Dataset(Xh)  # a fresh Dataset: validated and uploaded every call
            if world > 1:
                Zall = np.concatenate([Zh[i]] * world)  # every rank passes the full list; shards by rank
                depth_sharded(Zall, data, cfg)
            else:
                depth_batch_arrays(Zh[i], data, cfg, q0=q0s[i])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e2e_s = time.perf_counter() - t0
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=red_dev)
        if world > 1:
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * B * args.steps / float(tt.item()), "unit": "query-depths/s",
               "h2d_bytes_per_step": int(n * d * 8 + B * d * 8),
               "d2h_bytes_per_step": int(B * (8 + 8 * d + 8)),
               "api": "paper_2506_08262_b200.depth_batch_arrays -> rrs_depth_batch_host (C ABI)"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(X, notion, k, r, alpha)
            cpu["cpu_model"] = cpu_model()
        line = {
            "metric": "query-depths/s (RRS, all n points)", "value": value, "unit": "query-depths/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f16x2-split/f32-acc" if tensor else "f32",
            "data": "synthetic (reference generators: Toeplitz Gaussian / Student-t seed 0)",
            "config": {"workload": WORKLOAD_TEXT[wl], "notion": notion, "n": n, "d": d, "NRandom": k,
                       "n_refinements": r, "directions_per_refinement": m, "sphcap_shrink": alpha,
                       "queries_per_gpu_per_step": B, "global_batch": B * world, "parallelism": f"query-shard x{world}",
                       "dist_backend": args.dist_backend if world > 1 else None,
                       "l2": "flushed between timed steps (256 MiB write)",
                       "early_exit": bool(args.early_exit)},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "early_exit": early,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
