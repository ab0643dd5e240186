#!/usr/bin/env python
"""bench.py -- GANQ layer quantization (arxiv 2501.12956, Algorithm 1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2]

One step = the whole hot path for one layer: H = X X^T from the calibration tokens
(ganq_hessian), then ganq_quantize_layer (precondition, Cholesky, W H, K = 10 x {S-update,
T-update}).  Workload (BASELINE.json configs[1]): LLaMA-2-7B q_proj, W 4096 x 4096 fp32,
4-bit, X = 128 x 2048 = 262144 calibration tokens (bf16), K = 10; synthetic seeded data
(synthetic/, recipe in DESIGN.md).  Metric: rows*iter/s = m * K / layer time.

N > 1 (torchrun, one process per GPU, NCCL): tokens are sharded for H (whole
GANQ_HESSIAN_SUPERCHUNKs per rank), an exact integer all-reduce of the packed fixed-point
Hessian tiles (dist.py), rows sharded m/N per rank (strong scaling of one layer);
time = max over ranks of the CUDA-event time.

--impl reference runs the fp64 CPU oracle (oracle/, the only baseline this tier has) on a
bounded sample of the same workload and extrapolates to the layer (rank 0 only).
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

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic  # noqa: E402

METRIC = "4096x4096 4-bit layer quantize time (ms), rows·iter/s, % roofline @1/2/4/8"
UNIT = "rows*iter/s"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return dict(hbm_gbs=d.get("hbm_gbs", 6650.0), bf16=d.get("bf16_tflops", 1590.0),
                    bf16_sus=d.get("bf16_tflops_sustained", 1400.0), sm_mhz=d.get("sm_max_mhz", 1965.0),
                    source="measured")
    return dict(hbm_gbs=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_mhz=1965.0, source="fallback")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- oracle timing
ORACLE_ROWS = 64  # >= the host's cores (OpenMP over rows): every core has rows to solve


def oracle_sample(W_rows: np.ndarray, X_bits: np.ndarray, m: int, p: int, nbits: int, K: int):
    """One bounded sample of the layer on the fp64 oracle, the SAME sample in both arms.

    The sample is the share r/m of the layer that r of its m rows carry (rows are independent
    given H, Eq. 2): K x (S-step, T-step) on the r rows, H over r/m of the p tokens
    (X_bits holds p r / m tokens), and the full n x n preconditioned Cholesky, which cannot be
    split and is charged r/m of its measured time (it is a per-layer cost).  Every piece is timed
    (wall clock) in this call; value = r K / (t_H + t_ST + (r/m) t_chol) rows*iter/s, i.e. the
    layer throughput m K / (t_H m/r + t_ST m/r + t_chol) without any per-piece extrapolation
    beyond that proportional split.  Returns dict(value, wall_s, sample description, parts)."""
    import oracle
    oracle.build()
    ps, n = X_bits.shape
    r = W_rows.shape[0]
    t0 = time.perf_counter()
    H = oracle.hessian_bf16(X_bits)
    tH = time.perf_counter() - t0
    t0 = time.perf_counter()
    Hp, _ = oracle.precondition(H, "adaptive")
    L = oracle.cholesky(Hp)
    tC = time.perf_counter() - t0
    t0 = time.perf_counter()
    T = oracle.init_codebook(W_rows.astype(np.float32), nbits).astype(np.float64)
    for _ in range(K):
        Q, _ = oracle.sstep(W_rows, L, T)
        T = oracle.tstep(W_rows, Q, H, 1 << nbits)
    tR = time.perf_counter() - t0
    charged = tH + tR + tC * r / m
    return dict(value=r * K / charged, wall_s=tH + tC + tR, layer_s=charged * m / r,
                parts={"hessian_s": round(tH, 3), "cholesky_s": round(tC, 3), "s_t_steps_s": round(tR, 3)},
                sample=(f"oracle fp64 C (OpenMP, {cores()} threads): {r} of {m} rows x K={K} S+T iterations, "
                        f"H over {ps} of {p} tokens (the same {r}/{m} share), full {n}x{n} Cholesky charged "
                        f"{r}/{m} of its time; layer-equivalent {charged * m / r:.0f} s"))


def oracle_inputs(W_cpu: torch.Tensor, X: torch.Tensor, m: int, p: int, rows: int = ORACLE_ROWS):
    """The oracle sample's inputs: `rows` evenly spaced rows of W and the first p r / m tokens of X
    (bf16 bit patterns)."""
    r = min(rows, m)
    rows = np.linspace(0, m - 1, r).astype(int)
    ps = max(1, p * r // m)
    return W_cpu[rows].numpy().astype(np.float64), synthetic.bf16_bits(X[:ps])


def cores():
    v = os.environ.get("OMP_NUM_THREADS")
    return int(v) if v else (os.cpu_count() or 1)


# --------------------------------------------------------------------------- our arm
def choose_peaks(peaks, ck):
    """The roofline denominators: the BURST cuBLAS bf16 figure and the max SM clock, always.  A step
    mixes kernels of very different power (the dense Hessian and the fp64 Cholesky pull the clock
    down under `sw_power_cap`, the T-build runs near max), so the median clock of a capped run
    understates the clock of some stages (at c3 it produced fractions above 1); against the
    max-clock peaks every fraction is a lower bound.  The run's median clock is reported with it."""
    smax = ck.get("sm_max_mhz") or peaks["sm_mhz"]
    sm = ck.get("sm_mhz") or smax
    return dict(bf16=peaks["bf16"], clk_mhz=smax, hbm=peaks["hbm_gbs"],
                kind=f"burst at the max clock (run median {sm} MHz)", source=peaks["source"])


def stage_roofline(name, ms, launches, m, n, p, K, pk, nlev=16):
    """Algorithmic work of a stage per step against the peak of the unit that bounds it
    (SURVEY 8(d)).  Tensor peaks are derived from the measured bf16 figure by
    the nominal ratios of the profiling guide: tf32 = bf16 / 2, and an fp32-accurate tf32x3 product
    costs 3 tf32 passes.  The T-build (tgram) is bounded by FP32-ALU additions (SURVEY 8(d) G8:
    148 SM x 128 lanes x clock); its tensor-core one-hot formulation has its own ceiling
    (int8 = 2 x bf16 MAC/s, 3 digits x 2^N levels MACs per addition), reported beside it.
    fp64: 148 x 64 FMA lanes x 2 x clock.  Returns None for stages without a bound."""
    clk = pk["clk_mhz"] * 1e6
    fp64 = 148 * 64 * 2 * clk / 1e12
    tf32x3 = pk["bf16"] / 2 / 3
    alu_adds = 148 * 128 * clk / 1e12            # T additions/s
    s = ms / 1e3
    if s <= 0:
        return None
    extra = {}
    if name == "hessian":
        work, unit, bound, peak = n * (n + 1) * p / 1e12, "TFLOP/s", "tensor", pk["bf16"]
    elif name == "tgram":
        # the larger of SURVEY 8(d) G8's FP32-ALU bound (a CUDA-core T-build) and the ceiling of the
        # one-hot tensor-core formulation used here (the larger at 3 bits): never above 1
        form = 2 * pk["bf16"] / 2 / (3 * nlev)    # int8 MAC/s / (3 nlev MACs per addition)
        work, unit = K * m * n * (n - 1) / 2 / 1e12, "TFLOP/s"  # 1 addition = 1 flop
        bound, peak = ("alu", alu_adds) if alu_adds >= form else ("tensor", form)
        extra = {"formulation": "one-hot int8 tcgen05 (R-14)", "formulation_peak": round(form, 3),
                 "formulation_frac": round(work / s / form, 4)}
    elif name == "tsolve":
        work, unit, bound, peak = K * (5.0 * m * n + 4 * 8 * m * nlev * nlev) / 1e9, "GB/s", "hbm", pk["hbm"]
    elif name == "sstep":
        work, unit, bound, peak = K * m * n * (n - 1) / 1e12, "TFLOP/s", "tensor", tf32x3
    elif name == "gemm_wh":
        work, unit, bound, peak = 2.0 * m * n * n / 1e12, "TFLOP/s", "tensor", tf32x3
    elif name == "cholesky":
        work, unit, bound, peak = n ** 3 / 3 / 1e12, "TFLOP/s", "alu", fp64
    elif name == "precondition":
        work, unit, bound, peak = 2 * 8 * n * n / 1e9, "GB/s", "hbm", pk["hbm"]
    elif name == "derive_operands":
        work, unit, bound, peak = (8 + 8 + 4 + 4) * n * n / 1e9, "GB/s", "hbm", pk["hbm"]
    elif name == "init_codebook":
        work, unit, bound, peak = 4 * m * n / 1e9, "GB/s", "hbm", pk["hbm"]
    else:
        return None
    ach = work / s
    return dict(bound=bound, achieved=round(ach, 3), peak=round(peak, 3), unit=unit, frac=round(ach / peak, 4),
                ms=round(ms, 4), ideal_ms=round(1e3 * work / peak, 4), launches=int(launches), **extra)


def run_ours(args):
    from paper_2501_12956_b200 import _lib
    import paper_2501_12956_b200 as g
    from paper_2501_12956_b200.dist import shard_rows, shard_tokens
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    peaks = load_peaks()
    cfg = synthetic.CONFIGS[args.config]
    m, n, p, nbits, K = cfg["m"], cfg["n"], cfg["p"], cfg["nbits"], cfg["iters"]
    r0, r1 = shard_rows(m, world, rank)
    t0, t1 = shard_tokens(p, world, rank)
    W = synthetic.make_weights(m, n, seed=1000, device=dev)
    Xfull = synthetic.make_activations(p, n, seed=2000, device=dev)
    X = Xfull[t0:t1].contiguous()
    del Xfull
    Wl = W[r0:r1].contiguous()
    ml = r1 - r0
    H = torch.empty((n, n), dtype=torch.float64, device=dev)
    Q = torch.empty((ml, n), dtype=torch.uint8, device=dev)
    T = torch.empty((ml, 1 << nbits), dtype=torch.float32, device=dev)

    if world > 1:
        Pb, E = g.hessian_partials(X)  # buffers (sizes depend only on this rank's tokens)
        Hf = torch.empty(g.hessian_fixed_size(n), dtype=torch.int64, device=dev)

    def hessian_step(Xs):
        if world == 1:
            g.hessian(Xs, H=H)
        else:
            # exact fixed-point reduction (dist.py): MAX of the channel exponents, int64 SUM of the
            # packed lower-triangle tiles -> bitwise the single-GPU H
            g.hessian_partials(Xs, P=Pb, E=E)
            dist.all_reduce(E, op=dist.ReduceOp.MAX)
            g.hessian_fixed(Pb, Xs.shape[0], E, Hfix=Hf)
            dist.all_reduce(Hf)
            g.hessian_finalize(Hf, E, H=H)

    def step():
        hessian_step(X)
        g.quantize_layer(Wl, H, nbits, K, Q=Q, T=T)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    lib.ganq_profile_enable(1)
    n0 = int(lib.ganq_launch_count())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    launches = int(lib.ganq_launch_count()) - n0
    nst = 32  # >= GANQ_PROFILE_STAGES; ganq_profile_read returns the real count
    ms_arr = (ctypes_double_array(nst))
    ln_arr = (ctypes_int64_array(nst))
    nst = int(lib.ganq_profile_read(ms_arr, ln_arr, nst))
    lib.ganq_profile_enable(0)
    ck = clocks.stop()
    if world > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = m * K / (ms_step / 1e3)

    pk = choose_peaks(peaks, ck)
    stages = {}
    for i in range(nst):
        name = lib.ganq_profile_stage_name(i).decode()
        if ms_arr[i] <= 0:
            continue
        ms_i = ms_arr[i] / args.steps
        rl = stage_roofline(name, ms_i, ln_arr[i] / args.steps, ml, n, t1 - t0, K, pk, 1 << nbits)
        stages[name] = rl if rl else dict(ms=round(ms_i, 4), launches=int(ln_arr[i] / args.steps))
    dominant = max((k for k in stages if "frac" in stages[k]), key=lambda k: stages[k]["ms"])
    roof = {k: stages[dominant][k] for k in ("bound", "achieved", "peak", "unit", "frac")}
    roof["kernel"] = dominant
    roof["share_of_step"] = round(stages[dominant]["ms"] / ms_step, 4)
    roof["traffic"] = load_traffic(dominant)
    roof["peak_source"] = f"{pk['source']} ({pk['kind']}: bf16 {pk['bf16']:.1f} TF/s, clock {pk['clk_mhz']} MHz)"
    for k in ("formulation", "formulation_peak", "formulation_frac"):
        if k in stages[dominant]:
            roof[k] = stages[dominant][k]
    ideal = sum(v.get("ideal_ms", 0.0) for v in stages.values())
    layer_roof = {"ideal_ms": round(ideal, 4), "measured_ms": round(ms_step, 4), "frac": round(ideal / ms_step, 4),
                  "definition": "SURVEY 8(d): sum over stages of (algorithmic work / the peak of its bound) "
                                "divided by the measured layer time"}

    # ---- end to end through the public API with host buffers (pinned), H2D + D2H per step
    e2e = None
    if not args.no_e2e:
        # the public pipelined API (paper_2501_12956_b200.pipeline): every step uploads its X and W
        # from pinned host memory and downloads (Q, T); the upload of step k+1 overlaps step k's
        # solve (a user quantizing a sequence of layers); timed on the device from the first
        # upload to the last download
        from paper_2501_12956_b200.pipeline import LayerPipeline
        Xh = X.cpu().pin_memory()
        Wh = Wl.cpu().pin_memory()
        ks = max(2, args.steps)
        outs = [(torch.empty(Q.shape, dtype=Q.dtype).pin_memory(), torch.empty(T.shape, dtype=T.dtype).pin_memory())
                for _ in range(ks)]
        if world == 1:
            pipe = LayerPipeline(ml, n, X.shape[0], nbits, K, device=dev)
            pipe.run([(Wh, Xh)], outs[:1])  # warm-up
            pipe.finish()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(pipe.copy)
            pipe.run([(Wh, Xh)] * ks, outs)
            e1.record(pipe.copy)
            pipe.finish()
            te = e0.elapsed_time(e1) / ks
            api_name = "paper_2501_12956_b200.pipeline.LayerPipeline (upload of step k+1 overlaps step k)"
        else:
            # N > 1: each step uploads its token shard and rows, all-reduces H, solves, downloads
            Xd, Wd = torch.empty_like(X), torch.empty_like(Wl)
            Qh, Th = outs[0]

            def e2e_step():
                Xd.copy_(Xh, non_blocking=True)
                Wd.copy_(Wh, non_blocking=True)
                hessian_step(Xd)
                g.quantize_layer(Wd, H, nbits, K, Q=Q, T=T)
                Qh.copy_(Q, non_blocking=True)
                Th.copy_(T, non_blocking=True)
                torch.cuda.current_stream().synchronize()

            e2e_step()
            torch.cuda.synchronize()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(ks):
                e2e_step()
            e1.record()
            torch.cuda.synchronize()
            tt = torch.tensor([e0.elapsed_time(e1) / ks], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt.item())
            api_name = "paper_2501_12956_b200 fixed-point hessian + integer all_reduce + quantize_layer per step"
        e2e = {"value": round(m * K / (te / 1e3), 3), "unit": UNIT, "ms_per_step": round(te, 3),
               "h2d_bytes_per_step": int(Xh.numel() * Xh.element_size() + Wh.numel() * Wh.element_size()),
               "d2h_bytes_per_step": int(outs[0][0].numel() + outs[0][1].numel() * 4), "steps": ks,
               "api": api_name}

    # ---- NEXT-1: serving the layer's (Q, T) with the LUT GEMV vs an fp16 GEMV on W~ (cuBLAS)
    lut = None
    if rank == 0 and not args.no_lut:
        lut = lut_gemv_bench(g, Q, T, ml, n, nbits, peaks, dev)
        lut["outlier_split"] = outlier_bench(g, Wl, peaks)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Wr, Xs = oracle_inputs(W.cpu(), X, m, p)
        ob = oracle_sample(Wr, Xs, m, p, nbits, K)
        cpu = {"value": round(ob["value"], 4), "unit": UNIT, "cores": cores(), "kind": "oracle",
               "sample": ob["sample"], "wall_s": round(ob["wall_s"], 2), "parts": ob["parts"]}

    if rank == 0:
        out = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32+bf16+f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "m": m, "n": n, "n_bits": nbits,
                       "tokens": p, "iters": K, "rows_per_gpu": ml, "tokens_per_gpu": t1 - t0,
                       "parallelism": f"tokens+rows x{world}" if world > 1 else "single",
                       "l2": "inputs larger than L2 (X = 2.15 GB bf16 streamed every step)"},
            "layer_ms": round(ms_step, 4),
            "roofline": roof, "layer_roofline": layer_roof, "stages": stages, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
            "lut_gemv": lut,
            "clocks": ck,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def outlier_bench(g, W, peaks, reps=20, r=0.005):
    """NEXT-2: GANQ* split of the layer's W (Algorithm 2, r = 0.5 %), device time of the
    split + CSR kernels; algorithmic bytes = read W + write W_dense (+ the CSR)."""
    Wd, (off, col, val), _ = g.outlier_split(W, r)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.outlier_split(W, r)  # (synchronises once per call for the host nnz)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    nbytes = 2 * W.numel() * 4 + off.numel() * 8 + col.numel() * 8
    ach = nbytes / (us * 1e-6) / 1e9
    return {"us": round(us, 1), "nnz": int(col.numel()), "nnz_frac": round(col.numel() / W.numel(), 5),
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(ach / peaks["hbm_gbs"], 4)},
            "note": "includes the host synchronisation for nnz between the two kernels"}


def lut_gemv_bench(g, Q, T, m, n, nbits, peaks, dev, reps=200):
    """NEXT-1 (Fig. 1a): decode GEMV y = W~ x for the quantized layer, LUT kernel on the packed
    codes vs torch's fp16 GEMV (cuBLAS) on the dense fp16 W~.  Both rotate over copies whose
    total exceeds the 126 MB L2, so every call streams its weights from HBM."""
    P = g.pack_codes(Q, nbits)
    T16 = g.codebook_f16(T)
    W16 = torch.gather(T16, 1, Q.long())  # dense fp16 W~ for the baseline (dequantization path)
    x = torch.randn(1, n, dtype=torch.float16, device=dev)
    l2 = 126e6
    ncp = int(l2 // (P.numel() + T16.numel() * 2)) + 2
    Ps = [P.clone() for _ in range(ncp)]
    T16s = [T16.clone() for _ in range(ncp)]
    ncd = int(l2 // (W16.numel() * 2)) + 2
    Ws = [W16.clone() for _ in range(ncd)]
    y = torch.empty(1, m, dtype=torch.float32, device=dev)
    yd = torch.empty(1, m, dtype=torch.float16, device=dev)

    def timeit(fn, k):
        # the calls are captured in a CUDA graph: the GPU time of back-to-back kernels, no
        # host launch overhead (a Python call costs more than the kernel)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(k):
                fn(i)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for i in range(reps):
                fn(i % k)
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3  # us

    us_lut = timeit(lambda i: g.lut_gemm(Ps[i], T16s[i], x, n, Y=y), ncp)
    us_fp16 = timeit(lambda i: torch.matmul(x, Ws[i].t(), out=yd), ncd)
    lut_bytes = P.numel() + T16.numel() * 2 + x.numel() * 2 + m * 4
    fp16_bytes = W16.numel() * 2 + x.numel() * 2 + m * 2
    ach = lut_bytes / (us_lut * 1e-6) / 1e9
    return {"shape": f"{m}x{n}, {nbits}-bit, p = 1 (decode)", "lut_us": round(us_lut, 2),
            "fp16_cublas_us": round(us_fp16, 2), "speedup_vs_fp16": round(us_fp16 / us_lut, 3),
            "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(ach / peaks["hbm_gbs"], 4), "bytes_per_call": int(lut_bytes)},
            "fp16_achieved_gbs": round(fp16_bytes / (us_fp16 * 1e-6) / 1e9, 1),
            "l2": f"{ncp} / {ncd} rotating weight copies (> 126 MB L2)",
            "paper": "up to 2.57x end-to-end over FP16 on RTX 4090 (P:29) -- another machine and model"}


def ctypes_double_array(k):
    import ctypes
    return (ctypes.c_double * k)()


def ctypes_int64_array(k):
    import ctypes
    return (ctypes.c_int64 * k)()


def load_traffic(kernel):
    """dram read+write bytes per launch of `kernel` from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(path):
        return json.load(open(path)).get(kernel)
    return None


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle arm: every step is one oracle_sample() of the workload (the same sample as our
    arm's cpu_baseline), timed on the host cores; rank 0 only."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    cfg = synthetic.CONFIGS[args.config]
    m, n, p, nbits, K = cfg["m"], cfg["n"], cfg["p"], cfg["nbits"], cfg["iters"]
    W = synthetic.make_weights(m, n, seed=1000)
    # rows per step: the whole --steps K --warmup W run within about 200 s (the c2 sample costs
    # ~0.9 s of host time per row on 16 cores), never fewer rows than host cores
    r = min(m, ORACLE_ROWS, max(cores(), int(200.0 / max(1, args.steps + args.warmup) / 0.9)))
    X = synthetic.make_activations(max(1, p * r // m), n, seed=2000)
    Wr, Xs = oracle_inputs(W, X, m, p, rows=r)
    for _ in range(args.warmup):
        oracle_sample(Wr, Xs, m, p, nbits, K)
    vals, walls = [], []
    ob = None
    for _ in range(args.steps):
        ob = oracle_sample(Wr, Xs, m, p, nbits, K)
        vals.append(ob["value"])
        walls.append(ob["wall_s"])
    value = len(vals) / sum(1.0 / v for v in vals)  # units / total charged time
    out = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": int(os.environ.get("WORLD_SIZE", args.gpus)), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(walls) / len(walls), 1), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "m": m, "n": n, "n_bits": nbits, "tokens": p,
                   "iters": K, "sample": ob["sample"]},
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": cores(), "kind": "oracle",
                         "sample": ob["sample"], "parts": ob["parts"]},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "ms_per_step is the measured wall time of one oracle sample (see config.sample)",
    }
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None,
                    help="timed steps (default 20; 5 for --impl reference, whose steps are host oracle samples)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", choices=sorted(synthetic.CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-lut", action="store_true", help="skip the NEXT-1 LUT GEMV measurement")
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 5 if args.impl == "reference" else 20
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
