#!/usr/bin/env python
"""bench.py -- PrivFT encrypted fastText inference on B200 (BASELINE.json metric).

Default (N=1): one "step" = one ckks_privft_infer over a batch of B queries at the
PrivFT inference configuration (N = 2^13, L = 5 limbs (60 + 4x40 bits) + one
60-bit special prime, Delta = 2^40, vocabulary m = 500,000 -> K = 123 chunk ciphertexts per
query, embedding dim n = 300 (BASELINE "dim ~300"), c = 4 classes, polynomial softmax on).
It exercises every SURVEY 8(a) row: NTT/INTT (a1), limb-wise modular arithmetic (a2),
rescale (a3), key switching (a4), HMult+relin+rescale (a5, the softmax square), rotation
(a6) and TotalSum (a7), composed by the a8 sequence.  The first half of the BASELINE metric,
us per HMult+relin+rescale at N = 2^16 (l = 30), is measured in the same run and
reported under "hmult_n16".

Multi-GPU (torchrun): queries shard across ranks with no data-path collective ("weak"
scaling); value = all ranks' queries / max-over-ranks device time.

--impl reference times the oracle (oracle/, plain CPU RNS-CKKS written from the paper) on
a bounded sample of the same workload on this host's cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes

import numpy as np
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C4 = dict(log_n=13, limb_bits=[60, 40, 40, 40, 40], special_bits=60, scale=2.0 ** 40)
C3 = dict(log_n=16, limb_bits=[40] * 30, special_bits=60, scale=2.0 ** 40)
METRIC = "encrypted fastText inferences/sec"
HBM_PEAK_FALLBACK = 6534.5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=32, help="queries per GPU per step")
    ap.add_argument("--n", type=int, default=300, help="embedding dimension (BASELINE: ~300; paper: 50)")
    ap.add_argument("--classes", type=int, default=4)
    ap.add_argument("--m", type=int, default=500000, help="vocabulary size (P:441)")
    ap.add_argument("--no-poly", action="store_true", help="disable the polynomial softmax (A19)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-hmult", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the N = 2^12..2^16 op sweep")
    ap.add_argument("--no-matrix", action="store_true", help="skip the SURVEY 8(d) measurement matrix")
    ap.add_argument("--no-batches", action="store_true", help="skip the PrivFT batch / poly on-off sweep")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--hmult-iters", type=int, default=20)
    ap.add_argument("--cpu-cols", type=int, default=16, help="embedding columns in the oracle's bounded sample")
    ap.add_argument("--workload", choices=["infer", "train", "codec"], default="infer",
                    help="infer: PrivFT inference (default, BASELINE metric); train: one encrypted minibatch "
                         "training step (SURVEY C5 / row f1); codec: batched GPU encode+encrypt and "
                         "decrypt+decode of client vectors (row f4)")
    ap.add_argument("--vectors", type=int, default=1024, help="codec: slot vectors per GPU per step")
    ap.add_argument("--min-ms", type=float, default=0.0,
                    help="codec: raise --steps so the timed region lasts at least this long (clock sampling)")
    ap.add_argument("--examples", type=int, default=8, help="train: examples per GPU per minibatch")
    return ap.parse_args()


# ------------------------------------------------------------------------------ utils --
def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return HBM_PEAK_FALLBACK, "fallback"


def int_peak():
    """Integer roofline: Harvey/Shoup butterflies and 128-bit MACs per second with no memory
    traffic (bench/int_peak.cu), measured live; committed copy as fallback."""
    so = os.path.join(ROOT, "bench", "libintpeak.so")
    try:
        lib = ctypes.CDLL(so)
        out = (ctypes.c_double * 6)()
        if lib.int_peak(out) == 0:
            return dict(bfly_per_s=out[0], mac128_per_s=out[1], imad32_per_s=out[2], fbfly_per_s=out[4],
                        fmac_per_s=out[5], source="live")
    except OSError:
        pass
    d = json.load(open(os.path.join(ROOT, "bench", "peaks_int.json")))
    d["source"] = "committed bench/peaks_int.json"
    return d


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device, self.rows, self.proc = device, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 9:
                for nm, v in zip(names, r[5:9]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


# ------------------------------------------------------------------ oracle (CPU) arm --
_OS_ARGS = None


def _oracle_column(_):
    import oracle
    p, chunks, pts, gk = _OS_ARGS
    acc = None
    for ct, pt in zip(chunks, pts):
        x = oracle.mul_plain(p, ct, pt)
        acc = x if acc is None else oracle.add(p, acc, x)
    acc = oracle.rescale(p, acc)
    acc = oracle.total_sum(p, acc, gk)
    return oracle.rescale(p, oracle.mul_const(p, acc, 1.0 / 300, p.scale))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_sample(n_cols: int, m: int, seed: int = 0, cols: int = 16, workers: int = 1):
    """Bounded CPU sample of the same workload: `cols` embedding columns of ONE query
    through the oracle (per column: chunk-dot over all K chunks, rescale, TotalSum, x1/w,
    rescale), i.e. cols/n of a query's work; the output layer and softmax (< 1% of the
    work) are excluded.  workers > 1 runs the independent columns in forked processes (one
    oracle thread each).  Returns (seconds per query, description, threads, sample seconds)."""
    import multiprocessing as mp

    import oracle
    from paper_1908_06972_b200 import synth
    global _OS_ARGS
    p = oracle.preset("C4")
    t = p.slots
    K = -(-m // t)
    g = synth.rng(seed)
    rnd = lambda lv: [synth.uniform_residues(g, p.q[:lv], p.N) for _ in range(2)]
    chunks = [oracle.Ciphertext(rnd(p.L), p.L, p.scale) for _ in range(K)]
    pts = [oracle.Plaintext(synth.uniform_residues(g, p.q, p.N), p.L, p.scale) for _ in range(K)]
    kr = synth.KeyRandomness(seed, p.log_n, p.q, p.P)
    gk = {}
    for i in range(p.log_n - 1):  # keys are setup, not timed
        kappa, key = oracle.keygen_galois(p, kr.s, 1 << i, *kr.switch_key(1 + i))
        gk[kappa] = key
    cols = max(1, min(cols, n_cols))
    _OS_ARGS = (p, chunks, pts, gk)
    if workers > 1:
        with mp.get_context("fork").Pool(workers, initializer=oracle.worker_init) as pool:
            t0 = time.perf_counter()
            pool.map(_oracle_column, range(cols), chunksize=1)
            dt = time.perf_counter() - t0
        threads = workers
    else:
        t0 = time.perf_counter()
        for i in range(cols):
            _oracle_column(i)
        dt = time.perf_counter() - t0
        threads = int(os.environ.get("OMP_NUM_THREADS", 0)) or min(os.cpu_count() or 1, p.L)
    _OS_ARGS = None
    how = (f"{workers} forked processes x 1 thread, one column each" if workers > 1 else
           f"one process, OpenMP over <= {p.L} limbs")
    return dt * n_cols / cols, (f"{cols} of n={n_cols} embedding columns of 1 query at C4 (per column: K={K} "
                                f"chunk HMULPLAIN+HADD, rescale, TotalSum of {p.log_n - 1} rotations, x1/w, "
                                f"rescale) in {dt:.2f} s measured ({how}); per-query time = sample x n/{cols} "
                                f"(extrapolated)"), threads, dt


def cpu_baseline(n, m, cols):
    """The oracle on this host's cores: all cores (columns in parallel) and one core."""
    import oracle
    oracle.build()
    nproc = os.cpu_count() or 1
    cols_all = max(cols, nproc)
    dt, desc, threads, sample_s = oracle_sample(n, m, cols=cols_all, workers=nproc)
    out = {"value": 1.0 / dt, "unit": "inferences/s", "cores": threads, "kind": "oracle", "sample": desc,
           "seconds_per_query": dt, "sample_seconds": sample_s, "cpu_model": cpu_model(), "nproc": nproc}
    lib = oracle.lib()
    lib.or_set_threads(1)
    dt1, desc1, _, s1 = oracle_sample(n, m, cols=2, workers=1)
    lib.or_set_threads(nproc)
    out["one_core"] = {"value": 1.0 / dt1, "unit": "inferences/s", "cores": 1, "seconds_per_query": dt1,
                       "sample": desc1.replace("OpenMP over <= 5 limbs", "1 thread")}
    return out


def infer_config(args, world):
    """The inference workload's config (shared by both arms so the driver compares like for like)."""
    N, L = 1 << C4["log_n"], len(C4["limb_bits"])
    K = -(-args.m // (N // 2))
    B, poly = args.batch, not args.no_poly
    return {"workload": f"PrivFT encrypted inference C4: N=2^13, L=5 (60+4x40-bit) + 60-bit P, "
                        f"Delta=2^40, m={args.m} (K={K} chunks), n={args.n}, c={args.classes}, "
                        f"poly_softmax={poly}",
            "batch_per_gpu": B, "global_batch": B * world, "parallelism": f"query-sharded x{world}",
            "l2": "inputs larger than L2 (bag %.1f GB, H %.1f GB per GPU)" % (
                B * K * 2 * L * N * 8 / 1e9, args.n * K * L * N * 8 / 1e9)}


def run_reference(args, rank, world):
    """The oracle arm: each step is a bounded sample of the same workload (cols/n of one query)
    on all host cores; value = extrapolated inferences/s; ms_per_step = the measured sample."""
    if rank != 0:
        return
    import oracle
    oracle.build()
    nproc = os.cpu_count() or 1
    cols = max(args.cpu_cols, nproc)
    times, samples = [], []
    desc = ""
    threads = nproc
    for i in range(args.warmup + args.steps):
        dt, desc, threads, sample_s = oracle_sample(args.n, args.m, seed=i, cols=cols, workers=nproc)
        if i >= args.warmup:
            times.append(dt)
            samples.append(sample_s)
    per_query = statistics.mean(times)
    value = 1.0 / per_query
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "inferences/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(samples) * 1e3,
            "step_definition": f"one bounded sample = {cols}/{args.n} of one query's columns; value is "
                               f"extrapolated to whole queries (x {args.n}/{cols})",
            "extrapolated": True, "seconds_per_query_extrapolated": per_query,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (seeded uniform-residue ciphertexts/plaintexts of the C4 shapes)",
            "config": infer_config(args, world),
            "cpu_baseline": {"value": value, "unit": "inferences/s", "cores": threads, "kind": "oracle",
                             "sample": desc, "cpu_model": cpu_model()},
            "e2e": {"value": value, "unit": "inferences/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ GPU arm ------
def uniform_limbs(torch, shape_prefix, primes, N, device, gen):
    """uint64 residues (int64 view), uniform mod primes[i] on limb i: [*prefix, len(primes), N]."""
    t = torch.empty((*shape_prefix, len(primes), N), dtype=torch.int64, device=device)
    for i, q in enumerate(primes):
        t[..., i, :] = torch.randint(0, q, (*shape_prefix, N), dtype=torch.int64, device=device, generator=gen)
    return t


def gaussian(torch, shape, device, gen):
    return torch.clamp(torch.round(torch.randn(shape, device=device, generator=gen) * 3.2), -19, 19).to(torch.int64)


def setup_keys(torch, ctx, steps, gen):
    dev = ctx.device
    N, L = ctx.N, ctx.L
    s = torch.randint(0, 2, (N,), dtype=torch.int64, device=dev, generator=gen)
    ctx.set_secret(s)
    ctx.keygen_public(uniform_limbs(torch, (), ctx.q, N, dev, gen), gaussian(torch, (N,), dev, gen))
    ext, D = ctx.q + ctx.special, ctx.dnum
    ctx.keygen_relin(uniform_limbs(torch, (D,), ext, N, dev, gen), gaussian(torch, (D, N), dev, gen))
    for st in steps:
        ctx.keygen_galois(st, uniform_limbs(torch, (D,), ext, N, dev, gen), gaussian(torch, (D, N), dev, gen))


def bfly_equiv(v, peaks):
    """Work in integer-butterfly equivalents: each unit of work weighted by the time it takes
    at its own measured peak (integer butterflies, FP64-pipe butterflies, 128-bit integer MACs,
    FP64-pipe modular MACs)."""
    return (v["bfly"] + v.get("fbfly", 0.0) * peaks["bfly_per_s"] / peaks["fbfly_per_s"]
            + v["mac"] * peaks["bfly_per_s"] / peaks["mac128_per_s"]
            + v.get("fmac", 0.0) * peaks["bfly_per_s"] / peaks["fmac_per_s"])


def roofline_of(prof, peaks, hbm_peak, hbm_src):
    """Dominant kernel (largest device-time share) against the measured integer peak, or
    against measured HBM bandwidth when the kernel does no modular arithmetic (codec FFTs)."""
    tot = sum(v["ms"] for v in prof.values()) or 1.0
    name, v = max(prof.items(), key=lambda kv: kv[1]["ms"])
    traffic, traffic_src = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json"))).get(name)
        if tr:
            traffic = tr["dram_bytes"] / tr["algorithmic_bytes"] * v["bytes"] / max(v["launches"], 1)
            traffic_src = f"{tr['capture']} (dram/algorithmic = {tr['dram_bytes'] / tr['algorithmic_bytes']:.3f}, " \
                          f"scaled to this run's average launch)"
    except (OSError, ValueError, KeyError):
        pass
    bfly_eq = bfly_equiv(v, peaks)
    sec = v["ms"] * 1e-3
    achieved = bfly_eq / sec / 1e9
    peak = peaks["bfly_per_s"] / 1e9
    hbm = v["bytes"] / sec / 1e9
    if bfly_eq == 0:
        return {"kernel": name, "bound": "hbm", "achieved": hbm, "peak": hbm_peak, "unit": "GB/s",
                "frac": hbm / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                "share_of_step": v["ms"] / tot, "avg_launch_us": v["ms"] * 1e3 / max(v["launches"], 1),
                "work_per_launch": {"bytes": v["bytes"] / max(v["launches"], 1)}, "peak_source": hbm_src}
    return {"kernel": name, "bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gbfly/s",
            "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src, "share_of_step": v["ms"] / tot,
            "avg_launch_us": v["ms"] * 1e3 / max(v["launches"], 1),
            "work_per_launch": {"bfly": v["bfly"] / max(v["launches"], 1), "mac": v["mac"] / max(v["launches"], 1),
                                "fbfly": v.get("fbfly", 0.0) / max(v["launches"], 1),
                                "fmac": v.get("fmac", 0.0) / max(v["launches"], 1),
                                "bytes": v["bytes"] / max(v["launches"], 1)},
            "work_split": {"int_bfly": v["bfly"], "fp64_bfly": v.get("fbfly", 0.0), "mac": v["mac"],
                           "fp64_mac": v.get("fmac", 0.0)},
            "peak_source": f"bench/int_peak.cu ({peaks.get('source')}): 64-bit Harvey/Shoup butterflies/s on the "
                           f"integer pipe; FP64-pipe butterflies, 128-bit integer MACs and FP64-pipe modular MACs converted at their measured "
                           f"rates (achieved/peak = ideal time at the measured peaks / measured time)",
            "hbm_view": {"achieved_gbs": hbm, "peak_gbs": hbm_peak, "frac": hbm / hbm_peak, "peak_source": hbm_src}}


def hmult_c3(torch, ckks, dev, iters, hbm_peak, gen, alpha=1, K=1, sp_bits=None, peaks=None):
    """us per HMult+relin+rescale at N=2^16, l=30 (BASELINE metric, first half).
    alpha = K = 1: per-limb key switching (reading A6); otherwise hybrid with K
    special primes of sp_bits bits (40/41: FP64-mode special slots; 40: compact key rows, DESIGN 7)."""
    sp_bits = sp_bits or C3["special_bits"]
    ctx = ckks.Context(C3["log_n"], C3["limb_bits"], sp_bits, C3["scale"], device=dev.index or 0,
                       n_special=K, digit_limbs=alpha)
    N, L = ctx.N, ctx.L
    s = torch.randint(0, 2, (N,), dtype=torch.int64, device=dev, generator=gen)
    ctx.set_secret(s)
    ext, Dn = ctx.q + ctx.special, ctx.dnum
    ctx.keygen_relin(uniform_limbs(torch, (Dn,), ext, N, dev, gen), gaussian(torch, (Dn, N), dev, gen))
    torch.cuda.synchronize()
    A = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q, N, dev, gen), L, ctx.scale)
    B = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q, N, dev, gen), L, ctx.scale)
    T = ctx.alloc(1, 2, L)
    O = ctx.alloc(1, 2, L - 1)

    def fused():  # ckks_mul_relin_rescale: the one-call HMult+relin+rescale of the C ABI
        ctx.mul_relin_rescale(A, B, out=T)

    def two_calls():  # ckks_mul_relin, then ckks_rescale
        ctx.mul_relin(A, B, out=T)
        ctx.rescale(T, out=O)

    def timed(f):
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / iters

    us = timed(fused)
    us2 = timed(two_calls)
    us_graph = graph_us(torch, ctx, fused, iters)  # the same launch sequence replayed as one CUDA graph
    ctx.profile(True)  # per-kernel split: a second pass with CUDA events around every launch
    for _ in range(iters):
        fused()
    torch.cuda.synchronize()
    ctx.profile(False)
    prof = ctx.profile_read()
    l = L
    key_limbs = 2 * Dn * (l + K)
    alg_bytes = 8 * N * (4 * l + key_limbs + 2 * (l - 1))
    beta = -(-l // alpha)
    # limb NTTs of the one-call op: alpha = 1 (A6 + the A7 fused tail); hybrid: INTT(d2), ModUp
    # slots beta (l + K) - l, the fused ModDown + rescale tail's INTTs (K + 1 per polynomial) and
    # its broadcast NTT (l - 1 per polynomial)
    ntts = (l * l + 5 * l + 2) if (alpha == 1 and K == 1) else (l + beta * (l + K) - l + 2 * (K + 1) + 2 * (l - 1))
    out = {"us": us, "us_two_calls": us2, "us_graph": us_graph,
           "op": "ckks_mul_relin_rescale (us_two_calls: ckks_mul_relin + ckks_rescale; us_graph: one CUDA graph)",
           "config": f"N=2^16, l=30 x 40-bit, K={K} x {sp_bits}-bit special, alpha={alpha} (dnum={Dn})",
           "algorithmic_bytes": alg_bytes, "hbm_frac": alg_bytes / (us * 1e-6) / 1e9 / hbm_peak,
           "limb_ntts": ntts,
           "kernels_ms_per_op": {k: v["ms"] / iters for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])},
           "paper_v100_ms": 34.86}
    if peaks:  # composite ALU fraction: the op's butterflies / MACs at their measured peaks vs its time
        out["alu_frac"] = sum(bfly_equiv(v, peaks) for v in prof.values()) / iters / (us * 1e-6) / peaks["bfly_per_s"]
    ctx.close()
    return out


# N = 2^12 .. 2^16 sweep (north star: "throughput is reported at N = 2^12 through 2^16"):
# SURVEY Appendix C presets C1, C4, C2, C3 and a 16-limb 2^15 point between C2 and C3.
SWEEP = [("C1", 12, [30] * 3, 2.0 ** 30), ("C4", 13, [60, 40, 40, 40, 40], 2.0 ** 40),
         ("C2", 14, [40] * 8, 2.0 ** 40), ("N15", 15, [40] * 16, 2.0 ** 40), ("C3", 16, [40] * 30, 2.0 ** 40)]


def graph_us(torch, ctx, f, iters):
    """us per op when the op's launch sequence is captured once into a CUDA graph and replayed
    (the library is stream-ordered on its context stream, pointed at the capture stream)."""
    try:
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            ctx.set_stream(s)
            f()
        ctx.set_stream(torch.cuda.current_stream())
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1e3 / iters
    except Exception:  # capture is a measurement aid, never required
        ctx.set_stream(torch.cuda.current_stream())
        torch.cuda.synchronize()
        return None


def op_sweep(torch, ckks, dev, gen, hbm_peak, peaks, iters=10):
    """Per ring size: us per HMult+relin+rescale, per rotation (one key switch) and per limb-NTT
    pair (forward + inverse), at one ciphertext (latency) and at a batch of ~2^21 words per
    polynomial (throughput), each with its HBM fraction (the op's algorithmic bytes) and its
    composite ALU fraction (kernel work at the measured per-pipe peaks, as the roofline line)."""
    out = {}
    for name, log_n, bits, scale in SWEEP:
        ctx = ckks.Context(log_n, bits, 60, scale, device=dev.index or 0)
        N, L = ctx.N, ctx.L
        setup_keys(torch, ctx, [1], gen)
        key_limbs = 2 * ctx.dnum * (L + 1)
        rows = {"N": N, "limbs": L, "primes_bits": bits, "special_bits": 60}
        for count in sorted({1, max(1, (1 << 21) // (N * L))}):
            A = ckks.Buf(uniform_limbs(torch, (count, 2), ctx.q, N, dev, gen), L, ctx.scale)
            Bb = ckks.Buf(uniform_limbs(torch, (count, 2), ctx.q, N, dev, gen), L, ctx.scale)
            T, O, R = ctx.alloc(count, 2, L), ctx.alloc(count, 2, L - 1), ctx.alloc(count, 2, L)
            X = uniform_limbs(torch, (count * 2,), ctx.q, N, dev, gen)
            ops = {
                "hmult_relin_rescale": (lambda: ctx.mul_relin_rescale(A, Bb, out=T),
                                        8 * N * (4 * L * count + key_limbs + 2 * (L - 1) * count)),
                "rotate": (lambda: ctx.rotate(A, 1, out=R), 8 * N * (4 * L * count + key_limbs)),
                "ntt_fwd_inv": (lambda: (ctx.ntt(X), ctx.ntt(X, inverse=True)), 8 * N * 4 * 2 * L * count),
            }
            res = {}
            for op, (f, alg) in ops.items():
                for _ in range(2):
                    f()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(iters):
                    f()
                e1.record()
                torch.cuda.synchronize()
                sec = e0.elapsed_time(e1) * 1e-3 / iters
                ctx.profile(True)
                for _ in range(iters):
                    f()
                torch.cuda.synchronize()
                ctx.profile(False)
                prof = ctx.profile_read()
                eq = sum(bfly_equiv(v, peaks) for v in prof.values()) / iters
                res[op] = {"us_per_op": sec * 1e6 / count, "hbm_frac": alg / sec / 1e9 / hbm_peak,
                           "alu_frac": eq / sec / peaks["bfly_per_s"]}
                if count == 1:  # launch-bound at small N: the same op replayed as one CUDA graph
                    res[op]["us_per_op_graph"] = graph_us(torch, ctx, f, iters)
            rows[f"count_{count}"] = res
            del A, Bb, T, O, R, X
        ctx.close()
        torch.cuda.empty_cache()
        out[name] = rows
    return out


def naf_steps(steps: int, t: int) -> list[int]:
    """Signed power-of-two rotation keys the library applies for `steps` (reading A10): NAF
    digits of steps mod t (host bookkeeping for key setup; the library decomposes itself)."""
    s, out, i = steps % t, [], 0
    while s > 0:
        if s & 1:
            d = 2 - (s & 3)
            s -= d
            if (1 << i) < t:
                out.append(d * (1 << i))
        s >>= 1
        i += 1
    return out


def _time_op(torch, ctx, f, iters, peaks):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    sec = e0.elapsed_time(e1) * 1e-3 / iters
    ctx.profile(True)
    for _ in range(iters):
        f()
    torch.cuda.synchronize()
    ctx.profile(False)
    prof = ctx.profile_read()
    eq = sum(bfly_equiv(v, peaks) for v in prof.values()) / iters
    return sec, eq / sec / peaks["bfly_per_s"]


# Table 2, V100 ms, for context beside the matching rows
PAPER_T2 = {"(14,360)": {"hmul_rel": 0.74, "rescale": 0.14, "mulplain": 0.02, "addplain": 0.04, "rot_lhw": 0.88,
                         "rot_hhw": 6.09},
            "(16,1770)": {"hmul_rel": 33.58, "rescale": 1.28, "mulplain": 0.14, "addplain": 0.18, "rot_lhw": 39.91,
                          "rot_hhw": 324.90}}


def matrix(torch, ckks, dev, gen, hbm_peak, peaks, iters=5):
    """SURVEY 8(d) measurement matrix: C2 NTT batch sweep, C2 key switching at l in {8, 4} with
    the LHW/HHW rotations, C1 HHW rotation, C3 ops at levels {30, 20, 10} (us per op, HBM
    fraction of the op's algorithmic bytes, composite ALU fraction)."""
    W = 8
    out = {}
    hbm = lambda b, sec: b / sec / 1e9 / hbm_peak

    def row(sec, alu, alg):
        return {"us": sec * 1e6, "hbm_frac": hbm(alg, sec), "alu_frac": alu}

    # ---- C2: N = 2^14, 8 x 40-bit ------------------------------------------------------
    ctx = ckks.Context(14, [40] * 8, 60, 2.0 ** 40, device=dev.index or 0)
    N, L = ctx.N, ctx.L
    sweep = {}
    for B in (1, 16, 128, 1024):
        X = uniform_limbs(torch, (B,), ctx.q, N, dev, gen)
        r = {}
        for dirn, inv in (("fwd", False), ("inv", True)):
            sec, alu = _time_op(torch, ctx, lambda: ctx.ntt(X, inverse=inv), iters, peaks)
            r[dirn] = {"us": sec * 1e6, "limb_ntt_per_s": B * L / sec, "GBps": 2 * B * L * N * W / sec / 1e9,
                       "hbm_frac": hbm(2 * B * L * N * W, sec), "alu_frac": alu}
        sweep[f"B{B}"] = r
        del X
    out["c2_ntt_sweep"] = {"config": "N=2^14, 8 x 40-bit limbs, B polynomials x 8 limbs per launch", **sweep}
    ks = {}
    steps_hhw = 5461
    setup_keys(torch, ctx, sorted(set(naf_steps(1, N // 2) + naf_steps(steps_hhw, N // 2))), gen)
    for l in (8, 4):
        A = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q[:l], N, dev, gen), l, ctx.scale)
        Bb = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q[:l], N, dev, gen), l, ctx.scale)
        T, R = ctx.alloc(1, 2, l), ctx.alloc(1, 2, l)
        key_b = 2 * l * (l + 1)  # key limbs read: digits j < l, b and a, limbs q_0..q_{l-1}, P
        r = {}
        sec, alu = _time_op(torch, ctx, lambda: ctx.mul_relin(A, Bb, out=T), iters, peaks)
        r["mul_relin"] = row(sec, alu, N * W * (4 * l + key_b + 2 * l))
        sec, alu = _time_op(torch, ctx, lambda: ctx.rotate(A, 1, out=R), iters, peaks)
        r["rotate_lhw_1"] = row(sec, alu, N * W * (4 * l + key_b))
        nd = len(naf_steps(steps_hhw, N // 2))
        sec, alu = _time_op(torch, ctx, lambda: ctx.rotate(A, steps_hhw, out=R), iters, peaks)
        r[f"rotate_hhw_{steps_hhw}"] = row(sec, alu, nd * N * W * (4 * l + key_b))
        r[f"rotate_hhw_{steps_hhw}"]["naf_weight"] = nd
        r["hhw_over_lhw"] = r[f"rotate_hhw_{steps_hhw}"]["us"] / r["rotate_lhw_1"]["us"]
        ks[f"l{l}"] = r
        del A, Bb, T, R
    out["c2_keyswitch"] = {"config": "N=2^14, 8 x 40-bit + 60-bit P, alpha=1; relin / Galois keys at level 8",
                           "paper_v100_ms_(14,360)": PAPER_T2["(14,360)"], **ks}
    ctx.close()
    torch.cuda.empty_cache()
    # ---- C1: N = 2^12 HHW -------------------------------------------------------------
    ctx = ckks.Context(12, [30] * 3, 60, 2.0 ** 30, device=dev.index or 0)
    N, L = ctx.N, ctx.L
    setup_keys(torch, ctx, sorted(set(naf_steps(1, N // 2) + naf_steps(1365, N // 2))), gen)
    A = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q, N, dev, gen), L, ctx.scale)
    R = ctx.alloc(1, 2, L)
    r = {}
    for st in (1, 1365):
        sec, alu = _time_op(torch, ctx, lambda: ctx.rotate(A, st, out=R), iters, peaks)
        r[f"rotate_{st}"] = {"us": sec * 1e6, "alu_frac": alu, "naf_weight": len(naf_steps(st, N // 2))}
    r["hhw_over_lhw"] = r["rotate_1365"]["us"] / r["rotate_1"]["us"]
    out["c1_rotations"] = {"config": "N=2^12, 3 x 30-bit, single ciphertext (launch-bound)", **r}
    ctx.close()
    del A, R
    torch.cuda.empty_cache()
    # ---- C3: N = 2^16 at levels 30 / 20 / 10 ---------------------------------------------
    ctx = ckks.Context(C3["log_n"], C3["limb_bits"], C3["special_bits"], C3["scale"], device=dev.index or 0)
    N, L = ctx.N, ctx.L
    hhw = 21845
    setup_keys(torch, ctx, sorted(set(naf_steps(1, N // 2) + naf_steps(hhw, N // 2))), gen)
    lv = {}
    for l in (30, 20, 10):
        A = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q[:l], N, dev, gen), l, ctx.scale)
        Bb = ckks.Buf(uniform_limbs(torch, (1, 2), ctx.q[:l], N, dev, gen), l, ctx.scale)
        P_ = ckks.Buf(uniform_limbs(torch, (1, 1), ctx.q[:l], N, dev, gen), l, ctx.scale)
        T, O, R = ctx.alloc(1, 2, l), ctx.alloc(1, 2, l - 1), ctx.alloc(1, 2, l)
        key_b = 2 * l * (l + 1)
        r = {}
        sec, alu = _time_op(torch, ctx, lambda: ctx.mul_relin_rescale(A, Bb, out=T), iters, peaks)
        r["hmult_relin_rescale"] = row(sec, alu, N * W * (4 * l + key_b + 2 * (l - 1)))
        sec, alu = _time_op(torch, ctx, lambda: ctx.rescale(A, out=O), iters, peaks)
        r["rescale"] = row(sec, alu, N * W * (4 * l - 2))
        sec, alu = _time_op(torch, ctx, lambda: ctx.mul_plain(A, P_, out=R), iters, peaks)
        r["mul_plain"] = row(sec, alu, N * W * 5 * l)
        sec, alu = _time_op(torch, ctx, lambda: ctx.add(A, Bb, out=R), iters, peaks)
        r["add"] = row(sec, alu, N * W * 6 * l)
        sec, alu = _time_op(torch, ctx, lambda: ctx.rotate(A, 1, out=R), iters, peaks)
        r["rotate_lhw_1"] = row(sec, alu, N * W * (4 * l + key_b))
        if l == 30:
            nd = len(naf_steps(hhw, N // 2))
            sec, alu = _time_op(torch, ctx, lambda: ctx.rotate(A, hhw, out=R), 2, peaks)
            r[f"rotate_hhw_{hhw}"] = row(sec, alu, nd * N * W * (4 * l + key_b))
            r[f"rotate_hhw_{hhw}"]["naf_weight"] = nd
            r["hhw_over_lhw"] = r[f"rotate_hhw_{hhw}"]["us"] / r["rotate_lhw_1"]["us"]
        lv[f"l{l}"] = r
        del A, Bb, P_, T, O, R
    out["c3_levels"] = {"config": "N=2^16, 30 x 40-bit + 60-bit P, alpha=1, one ciphertext",
                        "paper_v100_ms_(16,1770)": PAPER_T2["(16,1770)"], **lv}
    ctx.close()
    torch.cuda.empty_cache()
    return out


def hmult_c3_sharded(torch, ckks, dev, iters, world, rank, pipelined=False):
    """us per HMult+relin+rescale at C3 with the RNS limbs sharded over the `world` ranks
    (north star): local digits -> NCCL all-gather -> ModUp / inner product /
    ModDown for the owned targets, then the sharded rescale (broadcast of the last limb).
    Device time, max over ranks.  Keys and inputs come from one seed on every rank."""
    import torch.distributed as dist
    from paper_1908_06972_b200 import dist as pdist
    ctx = ckks.Context(C3["log_n"], C3["limb_bits"], C3["special_bits"], C3["scale"], device=dev.index or 0)
    N, L = ctx.N, ctx.L
    g = torch.Generator(device=dev)
    g.manual_seed(4242)
    ctx.set_secret(torch.randint(0, 2, (N,), dtype=torch.int64, device=dev, generator=g))
    ext = ctx.q + ctx.special
    ctx.keygen_relin(uniform_limbs(torch, (ctx.dnum,), ext, N, dev, g), gaussian(torch, (ctx.dnum, N), dev, g))
    A_full = uniform_limbs(torch, (1, 2), ctx.q, N, dev, g)
    B_full = uniform_limbs(torch, (1, 2), ctx.q, N, dev, g)
    tr = pdist.Transport()
    lo, hi, w = pdist.limb_shard(L, world, rank)
    a = ckks.Buf(A_full[:, :, lo:hi].contiguous(), hi - lo, ctx.scale) if hi > lo else None
    b = ckks.Buf(B_full[:, :, lo:hi].contiguous(), hi - lo, ctx.scale) if hi > lo else None
    alloc = lambda cnt, nl: ctx.alloc(cnt, 2, nl)

    ksf = pdist.pipelined_sharded_keyswitch if pipelined else pdist.sharded_keyswitch

    def step():
        out = ksf(ctx, tr, 0, 0, a, b, L, L, alloc)
        return pdist.sharded_rescale(ctx, tr, out, L, L, 1, alloc)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) * 1e3 / iters], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ctx.close()
    return {"us": float(t.item()), "ranks": world, "limbs_per_rank": w,
            "config": "N=2^16, l=30 x 40-bit, alpha=1, limbs sharded over ranks (" +
                      ("per-rank NCCL broadcasts of the digit shards folded in as they land" if pipelined
                       else "NCCL all-gather of digits") + ")"}


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist

    from paper_1908_06972_b200 import build as libbuild
    from paper_1908_06972_b200 import ckks
    libbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hbm_peak, hbm_src = measured_peaks()
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    ctx = ckks.Context(C4["log_n"], C4["limb_bits"], C4["special_bits"], C4["scale"], device=local)
    N, L = ctx.N, ctx.L
    t = N // 2
    K = -(-args.m // t)
    B, n, c = args.batch, args.n, args.classes
    setup_keys(torch, ctx, [1 << i for i in range(ctx.log_n - 1)], gen)
    # model: NTT-form plaintexts of the packed H (n x K, level L) and O (n, level L-2)
    Hp = ckks.Buf(uniform_limbs(torch, (n * K, 1), ctx.q, N, dev, gen), L, ctx.scale)
    Op = ckks.Buf(uniform_limbs(torch, (n, 1), ctx.q[:L - 2], N, dev, gen), L - 2, ctx.scale)
    model = ctx.privft_model_wrap(Hp, Op, args.m, n, c)
    bag = ckks.Buf(uniform_limbs(torch, (B * K, 2), ctx.q, N, dev, gen), L, ctx.scale)
    w = torch.randint(50, 601, (B,), generator=torch.Generator().manual_seed(7 + rank)).numpy()
    poly = not args.no_poly
    out_level = L - 4 if poly else L - 3
    scores = ctx.alloc(B, 2, out_level, L - 3)
    step = lambda: ctx.privft_infer(model, bag, w, poly, out=scores)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n0 = ctx.launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - n0
    ms = e0.elapsed_time(e1)
    # per-kernel CUDA-event timing: the same K steps again with every launch bracketed by
    # events on the library stream (kept out of the headline pass: host-side event records
    # slow the enqueue of ~10^4 launches per step)
    ctx.profile(True)
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record()
    for _ in range(args.steps):
        step()
    p1.record()
    torch.cuda.synchronize()
    ctx.profile(False)
    prof = ctx.profile_read()
    prof_ms = p0.elapsed_time(p1)
    t_dev = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    ms_max = float(t_dev.item())
    value = B * world * args.steps / (ms_max * 1e-3)

    # e2e: through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        # ckks_privft_infer_host: every step uploads its bag from pinned host memory (on the
        # library's copy stream, overlapping the previous step's compute) and downloads its
        # scores; f0/f1 on the library stream bracket every copy and kernel of the K steps
        h_bag = torch.empty(bag.t.shape, dtype=torch.int64, pin_memory=True)
        h_bag.copy_(bag.t)
        h_out = torch.empty((B, 2, out_level, N), dtype=torch.int64, pin_memory=True)
        for _ in range(2):  # untimed: allocates both staging buffers
            ctx.privft_infer_host(model, h_bag, bag.scale, w, poly, h_out)
        ctx.sync()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e2e_steps = args.steps
        f0.record()
        for _ in range(e2e_steps):
            ctx.privft_infer_host(model, h_bag, bag.scale, w, poly, h_out)
        f1.record()
        ctx.sync()
        torch.cuda.synchronize()
        te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": B * world * e2e_steps / (float(te.item()) * 1e-3), "unit": "inferences/s",
               "h2d_bytes_per_step": h_bag.numel() * 8, "d2h_bytes_per_step": h_out.numel() * 8,
               "path": "pinned host bag -> ckks_privft_infer_host (upload overlapped with the previous step's "
                       "compute) -> pinned host scores"}
        del h_bag, h_out

    peaks = int_peak()
    roof = roofline_of(prof, peaks, hbm_peak, hbm_src)
    roof["measured_in"] = ("second pass of the same %d steps with CUDA events around every launch, kernels "
                           "serialised on one stream (ms_per_step there %.1f vs %.1f unprofiled, where the "
                           "integer- and FP64-class inner products share the SMs on two streams)"
                           % (args.steps, prof_ms / args.steps, ms / args.steps))
    tot_ms = sum(v["ms"] for v in prof.values())
    kernels = {k: {"share": v["ms"] / tot_ms, "launches": v["launches"]}
               for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
    pb = None
    if not args.no_batches and world == 1:
        # B in {1, 8, 64, 256} queries per step, poly softmax on and off,
        # with the paper's embedding dimension n = 50 (the first 50 columns of the bench
        # model); B = 1 with the softmax is the single-query latency
        del bag
        torch.cuda.empty_cache()
        n50 = min(50, n)
        m50 = ctx.privft_model_wrap(Hp.view(0, n50 * K), Op.view(0, n50), args.m, n50, c)
        pb = {"config": f"C4, m={args.m} (K={K}), n={n50} (paper), c={c}"}
        for Bx in (1, 8, 64, 256):
            bx = ckks.Buf(uniform_limbs(torch, (Bx * K, 2), ctx.q, N, dev, gen), L, ctx.scale)
            wx = torch.randint(50, 601, (Bx,), generator=torch.Generator().manual_seed(11 + Bx)).numpy()
            for pol in (True, False):
                ox = ctx.alloc(Bx, 2, L - 4 if pol else L - 3, L - 3)
                fx = lambda: ctx.privft_infer(m50, bx, wx, pol, out=ox)
                fx()
                torch.cuda.synchronize()
                reps = 3 if Bx <= 8 else 2
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    fx()
                e1.record()
                torch.cuda.synchronize()
                ms_x = e0.elapsed_time(e1) / reps
                pb[f"B{Bx}_{'poly' if pol else 'nopoly'}"] = {"ms_per_step": ms_x, "inferences_per_s": Bx / ms_x * 1e3,
                                                            "ms_per_query": ms_x / Bx}
                del ox
            del bx
            torch.cuda.empty_cache()
        pb["latency_B1_ms"] = pb["B1_poly"]["ms_per_step"]
        del m50
    else:
        del bag
    del model, scores, Hp, Op
    hm = None
    if not args.no_hmult:
        torch.cuda.empty_cache()
        ctx.close()
        hm = {"alpha1": hmult_c3(torch, ckks, dev, args.hmult_iters, hbm_peak, gen, peaks=peaks),
              "hybrid": hmult_c3(torch, ckks, dev, args.hmult_iters, hbm_peak, gen, alpha=10, K=10, sp_bits=40,
                                 peaks=peaks),
              "hybrid_k7_60bit": hmult_c3(torch, ckks, dev, args.hmult_iters, hbm_peak, gen, alpha=10, K=7,
                                          peaks=peaks)}
    if hm is not None and world > 1:
        try:
            hm["alpha1_limb_sharded"] = hmult_c3_sharded(torch, ckks, dev, args.hmult_iters, world, rank)
        except Exception as e:  # reported, never fatal
            hm["alpha1_limb_sharded"] = {"error": repr(e)}
        try:
            hm["alpha1_limb_sharded_pipelined"] = hmult_c3_sharded(torch, ckks, dev, args.hmult_iters, world, rank,
                                                                   pipelined=True)
        except Exception as e:  # reported, never fatal
            hm["alpha1_limb_sharded_pipelined"] = {"error": repr(e)}
    sweep = None
    if not args.no_sweep:
        sweep = op_sweep(torch, ckks, dev, gen, hbm_peak, peaks)
    mat = None
    if not args.no_matrix and world == 1:
        mat = matrix(torch, ckks, dev, gen, hbm_peak, peaks)
    cpu = None
    if rank == 0 and not args.no_cpu:
        try:
            cpu = cpu_baseline(n, args.m, args.cpu_cols)
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "error": repr(e)}
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    line = {"metric": METRIC, "value": value, "unit": "inferences/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic: seeded uniform-residue bag ciphertexts and NTT-form H/O plaintexts of the C4 "
                    "shapes; keys generated on device by libckks from seeded randomness",
            "config": infer_config(args, world),
            "clocks": clk.summary(), "e2e": e2e, "gpu_launches": launches, "roofline": roof,
            "cpu_baseline": cpu, "kernels": kernels, "hmult_n16": hm, "op_sweep": sweep, "matrix": mat,
            "privft_batches": pb, "int_peak": peaks}
    print(json.dumps(line), flush=True)


def run_train(args, rank, world, local):
    """One encrypted minibatch step of Alg "GDMiniBatchTraining" (row f1): N = 2^16,
    30 x 40-bit limbs, hybrid key switching (alpha = 10, K = 10 x 40-bit), m = 32768 (one
    chunk), n = 50, c = 2, E examples per GPU; gradients summed across ranks by all-gather +
    ckks_modadd_gathered, then the update.  Metric: seconds per minibatch step."""
    import torch
    import torch.distributed as dist

    from paper_1908_06972_b200 import build as libbuild
    from paper_1908_06972_b200 import ckks
    from paper_1908_06972_b200.dist import Transport
    libbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(99 + rank)
    ctx = ckks.Context(C3["log_n"], C3["limb_bits"], 40, C3["scale"], device=local, n_special=10,
                       digit_limbs=10)
    N, L = ctx.N, ctx.L
    n, c, E = min(args.n, 50), 2, args.examples
    setup_keys(torch, ctx, [1 << i for i in range(ctx.log_n - 1)], gen)
    H = ckks.Buf(uniform_limbs(torch, (n, 2), ctx.q, N, dev, gen), L, ctx.scale)
    O = ckks.Buf(uniform_limbs(torch, (n, 2), ctx.q, N, dev, gen), L, ctx.scale)
    bags = ckks.Buf(uniform_limbs(torch, (E, 2), ctx.q, N, dev, gen), L, ctx.scale)
    gs, gl = ctx.privft_train_plan(H, O, bags)
    t = N // 2
    y = [e % c for e in range(E)]
    w = [100 + e for e in range(E)]
    neg = ctx.alloc(E, 1, gl)
    for e in range(E):
        z = np.zeros(t)
        z[y[e]] = -1.0
        pt = ctx.encode(z, level=gl, scale=gs)
        neg.t[e].copy_(pt.t[0])
    neg.scale, neg.level = gs, gl
    mz = np.zeros(t)
    mz[:c] = 1.0
    mask = ctx.encode(mz, level=gl, scale=ctx.scale)
    tr = Transport() if world > 1 else None

    def step():
        GH, GO = ctx.privft_train_grad(H, O, bags, w, y, c, neg, mask)
        if tr is not None:  # cross-rank gradient sum: all-gather + modular add (NCCL cannot reduce mod q_i)
            for G in (GH, GO):
                g = tr.all_gather(G.t)
                ctx.modadd_gathered(g, world, G)
        return ctx.privft_train_update(H, O, GH, GO, 0.01)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n0 = ctx.launches()
    with Clocks(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
    t_dev = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    if rank != 0:
        return
    ms = float(t_dev.item()) / args.steps
    line = {"metric": "seconds per encrypted minibatch training step", "value": ms / 1e3, "unit": "s/step",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic uniform-residue model/bag ciphertexts of the C5 shapes",
            "config": {"workload": f"PrivFT encrypted training step (f1): N=2^16, 30x40-bit, hybrid alpha=10 K=10x40-bit, "
                                   f"m=32768, n={n}, c={c}, {E} examples/GPU, {E * world} per minibatch",
                       "examples_per_gpu": E, "parallelism": f"example-sharded x{world}, gradient all-gather+modadd"},
            "clocks": clk.summary(), "gpu_launches": ctx.launches() - n0,
            "paper": "8xV100: 5.04 days for 5 minibatches of 1,007,500 tokens (P:489), context only"}
    print(json.dumps(line), flush=True)


def run_codec(args, rank, world, local):
    """Row f4: the client side of P:272 on the GPU.  One step = V slot vectors (C4: N = 2^13,
    4096 complex slots, L = 5) through ckks_encode_batch -> ckks_encrypt -> ckks_decrypt ->
    ckks_decode_batch; vectors shard across ranks (weak scaling, no collective).
    Metric: vectors per second through the round trip."""
    import torch
    import torch.distributed as dist

    from paper_1908_06972_b200 import build as libbuild
    from paper_1908_06972_b200 import ckks
    libbuild.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    hbm_peak, hbm_src = measured_peaks()
    gen = torch.Generator(device=dev)
    gen.manual_seed(4321 + rank)
    ctx = ckks.Context(C4["log_n"], C4["limb_bits"], C4["special_bits"], C4["scale"], device=local)
    N, L, V = ctx.N, ctx.L, args.vectors
    setup_keys(torch, ctx, [], gen)
    z = torch.complex(torch.rand((V, N // 2), dtype=torch.float64, device=dev, generator=gen) * 2 - 1,
                      torch.rand((V, N // 2), dtype=torch.float64, device=dev, generator=gen) * 2 - 1)
    u = torch.randint(0, 2, (V, N), dtype=torch.int64, device=dev, generator=gen)
    e0, e1 = gaussian(torch, (V, N), dev, gen), gaussian(torch, (V, N), dev, gen)
    pt, ct, dec = ctx.alloc(V, 1, L), ctx.alloc(V, 2, L), ctx.alloc(V, 1, L)
    zo = torch.empty_like(z)
    lib = ckks.lib()

    def step():
        ctx.encode_batch(z, out=pt)
        pb, cb, db = pt.c(), ct.c(), dec.c()
        ctx._chk(lib.ckks_encrypt(ctx.h, ctypes.byref(pb), ckks._ptr(u), ckks._ptr(e0), ckks._ptr(e1),
                                  ctypes.byref(cb)), "ckks_encrypt")
        ctx._chk(lib.ckks_decrypt(ctx.h, ctypes.byref(cb), ctypes.byref(db)), "ckks_decrypt")
        ctx.decode_batch(dec.sync(db), out=zo)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    err = float((zo - z).abs().max())
    if args.min_ms > 0:  # size K so nvidia-smi sees the load (one probe step, untimed)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record()
        step()
        p1.record()
        torch.cuda.synchronize()
        need = math.ceil(args.min_ms / max(p0.elapsed_time(p1), 1e-3))
        t_need = torch.tensor([need], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t_need, op=dist.ReduceOp.MAX)
        args.steps = max(args.steps, int(t_need.item()))
    if world > 1:
        dist.barrier()
    n0 = ctx.launches()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        t0.record()
        for _ in range(args.steps):
            step()
        t1.record()
        torch.cuda.synchronize()
    launches = ctx.launches() - n0
    ms = t0.elapsed_time(t1)
    ctx.profile(True)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    ctx.profile(False)
    prof = ctx.profile_read()
    # e2e: pinned host vectors in, decoded host vectors out
    hz = torch.empty(z.shape, dtype=z.dtype, pin_memory=True)
    hz.copy_(z)
    ho = torch.empty(z.shape, dtype=z.dtype, pin_memory=True)
    torch.cuda.synchronize()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(args.steps):
        z.copy_(hz, non_blocking=True)
        step()
        ho.copy_(zo, non_blocking=True)
    f1.record()
    torch.cuda.synchronize()
    t_dev = torch.tensor([ms, f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
        dist.destroy_process_group()
    if rank != 0:
        return
    ms_max, fe = float(t_dev[0]), float(t_dev[1])
    tot_ms = sum(v["ms"] for v in prof.values())
    line = {"metric": "client vectors/s (encode+encrypt+decrypt+decode)", "value": V * world * args.steps / (ms_max * 1e-3),
            "unit": "vectors/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64+u64",
            "data": "synthetic: seeded uniform complex slot vectors in [-1,1]^2, binary u, Gaussian e0/e1",
            "config": {"workload": f"f4 client codec C4: N=2^13, L=5, {N // 2} complex slots, {V} vectors/GPU/step",
                       "l2": "inputs larger than L2 (%.0f MB of vectors + %.0f MB ciphertexts per step)" % (
                           V * N // 2 * 16 / 1e6, V * 2 * L * N * 8 / 1e6)},
            "max_abs_roundtrip_error": err, "clocks": clk.summary(),
            "e2e": {"value": V * world * args.steps / (fe * 1e-3), "unit": "vectors/s",
                    "h2d_bytes_per_step": hz.numel() * 16, "d2h_bytes_per_step": ho.numel() * 16},
            "gpu_launches": launches, "roofline": roofline_of(prof, int_peak(), hbm_peak, hbm_src),
            "kernels": {k: {"share": v["ms"] / tot_ms, "us_per_step": v["ms"] * 1e3 / args.steps,
                            "GBps": v["bytes"] / (v["ms"] * 1e-3) / 1e9}
                        for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}}
    print(json.dumps(line), flush=True)


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this script under torch.distributed.run
    with N ranks (one per GPU) on 127.0.0.1; rank 0 prints the JSON line.  NCCL INIT logging on."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    args = parse()
    rank, world, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: launch one rank per GPU")
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "train":
        run_train(args, rank, world, local)
    elif args.workload == "codec":
        run_codec(args, rank, world, local)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
