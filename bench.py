#!/usr/bin/env python
"""bench.py -- HyPHEN hot-path benchmark on B200 (BASELINE.json config 2).

Workload (BASELINE.json configs[1]): HRot / key-switch microbenchmark at
N = 2^16 over the full limb chain of Set_hyp (L+1 = 24, dnum = 6, K = 4;
P:1207-1208): one step = a batch of 64 non-hoisted rotations, ct_i rotated by
r_i = i + 1 with its own evaluation key (64 x 126 MiB of 6-byte-packed keys,
168 MB each unpacked as in P:1208, resident in HBM and larger than L2, so no
flush is needed).  The hoisted batch (ct_0 rotated by
1..64 with one shared ModUp) is reported alongside.

Metric: key switches per second (whole job, all ranks).  Multi-GPU: every rank
runs its own independent batch (weak scaling, no data-path collective);
timing is the max over ranks of the device time between barriers.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the CPU oracle (oracle/, test infrastructure) on the
host cores as the reference arm; rank 0 only.
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

import synth  # noqa: E402

BATCH = 64
E2E_CHUNK = 8  # rotations per e2e pipeline chunk
LEVEL = 23  # full chain: L+1 = 24 limbs
METRIC = "HRot keyswitch/s at N=2^16 (HBM GB/s vs peak); ResNet-20 conv-layer ms at 1/2/4/8 GPU"
UNIT = "keyswitch/s"
N = 1 << 16


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "fallback": True}


# --------------------------------------------------------------------------- ncu traffic
def ncu_traffic(fam_name):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the family's kernel, from the committed
    `ncu --set full` capture summary (profiles/ncu_traffic.json, written by tools/ncu_round.py), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
    except OSError:
        return None
    e = t.get("families", {}).get(fam_name)
    return None if e is None else {"bytes_per_launch": e["dram_bytes"], "kernel": e["kernel"],
                                   "items_per_launch": e.get("items"), "source": t.get("source")}


def traffic_fields(fam_name):
    """roofline.traffic = dram read + write bytes per launch (a number, or None) and where it comes from."""
    t = ncu_traffic(fam_name)
    return {"traffic": None if t is None else t["bytes_per_launch"], "traffic_detail": t}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        loaded = [s for s in sm if smax and s > 0.5 * max(smax)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(rows)}


# --------------------------------------------------------------------------- distributed
def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        # HY_DIST_BACKEND=gloo: a functional check of the multi-rank paths with several ranks sharing one
        # GPU (NCCL needs one GPU per rank); timings of such a run are not bench numbers
        backend = os.environ.get("HY_DIST_BACKEND", "nccl")
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------------------- CPU oracle timing
def oracle_keyswitch_rate(n_rot: int, level: int = LEVEL, seed: int = 0):
    """Time the CPU oracle's plain HRot at Set_hyp, on n_rot rotations (bounded sample).
    Key material is seeded uniform residues: the oracle's work is data-independent."""
    import oracle
    o = oracle.Oracle(**synth.PARAMS["hyp"])
    chain_all = list(range(o.nq + o.np_))
    evk = synth.residues(seed, (o.dnum * 2, len(chain_all), o.N), [int(o.moduli[t]) for t in chain_all]) \
        .reshape(o.dnum, 2, len(chain_all), o.N)
    ct = synth.residues(seed + 1, (2, level + 1, o.N), o.q[: level + 1])
    c = oracle.Ct(ct, level, 2.0**42)
    t0 = time.perf_counter()
    for i in range(n_rot):
        o.hrot(c, evk, i + 1)
    dt = time.perf_counter() - t0
    return n_rot / dt, dt


def oracle_conv_layer_extrapolated(name="L2_ds"):
    """ResNet-18 layer on the CPU oracle (too slow to run whole): time output 0, then outputs
    {0, 1}; the difference is the per-output cost, the rest the shared Slide_f, and the layer time is extrapolated
    linearly in n_o.  Data-independent work on seeded residues, as in oracle_conv_layers."""
    import oracle
    from oracle import hyphen as H
    o = oracle.Oracle(**synth.PARAMS["hyp"])
    chain_all = list(range(o.nq + o.np_))
    evk = synth.residues(7, (o.dnum * 2, len(chain_all), o.N), [int(o.moduli[t]) for t in chain_all]) \
        .reshape(o.dnum, 2, len(chain_all), o.N)

    class AnyKey(dict):
        def __missing__(self, r):
            return evk

    sp_t = {nm: sp for nm, sp, _ in R18_LAYERS}[name]
    sp = H.ConvSpec(*sp_t[:10], S=sp_t[10] if len(sp_t) > 10 else 1)
    K = synth.conv_weight(3000, sp.co, sp.ci, sp.f)
    plan = H.plan_caconv(sp, K) if sp.algo == "CA" else H.plan_raconv(sp, K)
    level = CA_LEVEL if sp.algo == "CA" else RA_LEVEL
    pts = {}

    def encode(v, lv):
        if lv not in pts:
            pts[lv] = oracle.Pt(synth.residues(8 + lv, (lv + 1, o.N), o.q[: lv + 1]), lv, float(o.q[lv]))
        return pts[lv]

    cts = [oracle.Ct(synth.residues(100 + i, (2, level + 1, o.N), o.q[: level + 1]), level, 2.0**42)
           for i in range(plan.n_in)]
    times = []
    for outs in ([0], [0, 1]):
        enc = H.EncConv(o, plan, AnyKey())
        enc.encode = encode
        t0 = time.perf_counter()
        enc.run(cts, outs)
        times.append(time.perf_counter() - t0)
    per_out = max(times[1] - times[0], 0.0)
    shared = max(times[0] - per_out, 0.0)
    return {"layer": f"ResNet-18 {name}", "n_out": plan.n_out, "oracle_ms_measured": [1000 * t for t in times],
            "oracle_ms_extrapolated": 1000 * (shared + plan.n_out * per_out), "level_in": level,
            "method": "outputs {0} and {0, 1} timed; layer = shared Slide_f + n_o x per-output (extrapolated)"}


def oracle_conv_layers(names=("L1_ca", "L1_ra")):
    """Time the CPU oracle's encrypted execution (oracle/hyphen.py EncConv, the plain C RNS-CKKS underneath) of
    whole ResNet-20 layers at the bench's levels, all outputs, on the host cores.  The oracle's work is
    data-independent, so keys, input ciphertexts and weight plaintexts are seeded uniform residues (one key
    serves every rotation amount; encoding is untimed in the paper, and is skipped)."""
    import oracle
    from oracle import hyphen as H
    o = oracle.Oracle(**synth.PARAMS["hyp"])
    chain_all = list(range(o.nq + o.np_))
    evk = synth.residues(7, (o.dnum * 2, len(chain_all), o.N), [int(o.moduli[t]) for t in chain_all]) \
        .reshape(o.dnum, 2, len(chain_all), o.N)

    class AnyKey(dict):
        def __missing__(self, r):
            return evk

    spec_of = {nm: sp for nm, sp, _ in R20_LAYERS}
    out = {}
    for li, nm in enumerate(names):
        sp = H.ConvSpec(*spec_of[nm][:10])
        K = synth.conv_weight(2000 + li, sp.co, sp.ci, sp.f)
        plan = H.plan_caconv(sp, K) if sp.algo == "CA" else H.plan_raconv(sp, K)
        level = CA_LEVEL if sp.algo == "CA" else RA_LEVEL
        enc = H.EncConv(o, plan, AnyKey())
        pts = {}

        def encode(v, lv, pts=pts):
            if lv not in pts:
                pts[lv] = oracle.Pt(synth.residues(8 + lv, (lv + 1, o.N), o.q[: lv + 1]), lv, float(o.q[lv]))
            return pts[lv]

        enc.encode = encode
        cts = [oracle.Ct(synth.residues(100 + i, (2, level + 1, o.N), o.q[: level + 1]), level, 2.0**42)
               for i in range(plan.n_in)]
        t0 = time.perf_counter()
        enc.run(cts)
        out[nm] = {"oracle_ms": 1000.0 * (time.perf_counter() - t0), "level_in": level, "n_out": plan.n_out,
                   "rotations": dict(plan.counts)}
    return out


def run_reference(args, ws, rank):
    """Reference arm: the CPU oracle as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    # all host cores (torchrun sets OMP_NUM_THREADS=1 per rank; the oracle's OpenMP reads it when it loads, below)
    cores = os.cpu_count()
    os.environ["OMP_NUM_THREADS"] = str(cores)
    # warm-up (untimed) and K timed steps, each step = 1 plain HRot at full level (bounded sample)
    for _ in range(args.warmup):
        oracle_keyswitch_rate(1)
    times = []
    for s in range(args.steps):
        rate, dt = oracle_keyswitch_rate(1, seed=s)
        times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = 1000.0 / ms
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": "C2 HRot keyswitch, N=2^16, Set_hyp L+1=24 dnum=6 K=4, plain (non-hoisted)",
                   "sample": "1 plain HRot at full level per step (of the 64-rotation batch)",
                   "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": "1 plain HRot per step, full level, OpenMP over limbs"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- ResNet-20 conv layers
# (name, (ci, co, w, f, stride, wp, gap, m, d, algo), multiplicity in ResNet-20): tb:resnet 20 parameter
# (P:1045-1050), Optimal (m, d) plan (1,2)/(2,4)/(4,8), DESIGN R-LAYOUT / R-DSCONV.
R20_LAYERS = [
    ("stem", (3, 16, 32, 3, 1, 32, 1, 1, 2, "CA"), 1),
    ("L1_ca", (16, 16, 32, 3, 1, 32, 1, 1, 2, "CA"), 3),
    ("L1_ra", (16, 16, 32, 3, 1, 32, 1, 2, 1, "RA"), 3),
    ("L2_ds", (16, 32, 32, 3, 2, 32, 1, 1, 2, "CA"), 1),
    ("L2_pconv", (16, 32, 32, 1, 2, 32, 1, 1, 2, "CA"), 1),
    ("L2_ca", (32, 32, 16, 3, 1, 32, 2, 2, 4, "CA"), 2),
    ("L2_ra", (32, 32, 16, 3, 1, 32, 2, 4, 2, "RA"), 3),
    ("L3_ds", (32, 64, 16, 3, 2, 32, 2, 2, 4, "CA"), 1),
    ("L3_pconv", (32, 64, 16, 1, 2, 32, 2, 2, 4, "CA"), 1),
    ("L3_ca", (64, 64, 8, 3, 1, 32, 4, 4, 8, "CA"), 2),
    ("L3_ra", (64, 64, 8, 3, 1, 32, 4, 8, 4, "RA"), 3),
]
CA_LEVEL, RA_LEVEL = 9, 6  # l+1 = 10 / 7 limbs (DESIGN R-LEVELS)

# ResNet-18 ImageNet stride-1 conv layers with PRCR |S| = 8, plan (1,1)/(2,2)/(4,4)/(8,8)
# (P:1164), widths 56/28/14/7 padded to 64/32/16/8 per gap (W_p = 64).  Multiplicity = 3x3 convs of each type.
R18_LAYERS = [
    ("L1_ca", (64, 64, 56, 3, 1, 64, 1, 1, 1, "CA", 8), 2),
    ("L1_ra", (64, 64, 56, 3, 1, 64, 1, 1, 1, "RA", 8), 2),
    ("L2_ca", (128, 128, 28, 3, 1, 64, 2, 2, 2, "CA", 8), 1),
    ("L2_ra", (128, 128, 28, 3, 1, 64, 2, 2, 2, "RA", 8), 2),
    ("L3_ca", (256, 256, 14, 3, 1, 64, 4, 4, 4, "CA", 8), 1),
    ("L3_ra", (256, 256, 14, 3, 1, 64, 4, 4, 4, "RA", 8), 2),
    ("L4_ca", (512, 512, 7, 3, 1, 64, 8, 8, 8, "CA", 8), 1),
    ("L4_ra", (512, 512, 7, 3, 1, 64, 8, 8, 8, "RA", 8), 2),
    # downsampling blocks: stride-2 dsconv and the 1x1 stride-2 shortcut (pconv), full (non-PRCR) weights
    # (PRCR needs stride 1, DESIGN R-PRCR); output RA(2d, 2m) at gap 2g feeds the next stage (R-DSCONV)
    ("L2_ds", (64, 128, 56, 3, 2, 64, 1, 1, 1, "CA", 1), 1),
    ("L2_pconv", (64, 128, 56, 1, 2, 64, 1, 1, 1, "CA", 1), 1),
    ("L3_ds", (128, 256, 28, 3, 2, 64, 2, 2, 2, "CA", 1), 1),
    ("L3_pconv", (128, 256, 28, 1, 2, 64, 2, 2, 2, "CA", 1), 1),
    ("L4_ds", (256, 512, 14, 3, 2, 64, 4, 4, 4, "CA", 1), 1),
    ("L4_pconv", (256, 512, 14, 1, 2, 64, 4, 4, 4, "CA", 1), 1),
]


def ks_fp64_ops(level: int, variant: str, alpha: int = 4, kp: int = 4) -> float:
    """FP64-pipe operations of one key switch at `level` in this implementation's algorithm (DESIGN.md section 5
    op counting: an NTT pass = 8 stages x N/2 butterflies x 8 ops, a BConv word 7a+2, an IP MAC 7 ops).
    variant: plain | hoisted (per rotation, the shared ModUp excluded) | modup (the shared ModUp of a hoisted
    group) | lazy_term (ModUp + IP of one HRotSum term) | moddown (one ModDown with its epilogue)."""
    n = level + 1
    E = n + kp
    P = 8 * (N // 2) * 8
    digits = [min(alpha, n - j * alpha) for j in range((n + alpha - 1) // alpha)]
    beta = len(digits)
    modup = n * P + n * P + sum((E - a) * (P + (7 * a + 2) * N) for a in digits)    # iNTT rows+cols, BConv, NTT cols
    modup_rows = sum((E - a) * P for a in digits)                                   # the digits' NTT row passes
    ip = 2 * beta * E * 7 * N
    moddown = 2 * kp * P + 2 * (kp * P + n * (P + (7 * kp + 2) * N)) + 2 * n * (P + 4 * N)
    if variant == "plain":
        return modup + modup_rows + ip + moddown
    if variant == "hoisted":
        return ip + moddown
    if variant == "modup":
        return modup + modup_rows
    if variant == "lazy_term":
        return modup + modup_rows + ip
    if variant == "moddown":
        return moddown
    raise ValueError(variant)


NVLINK_GBS = 700.0  # measured all-gather / peer-copy class bandwidth per direction (B200_PROFILING.md: 725-770 GB/s)


def scaling_model(p, algo: str, level: int, ms: float, hoisted_rate: float, plain_rate: float):
    """Per-rank cost model of a conv layer on G GPUs from its measured 1-GPU time:
    t_G = t_repeated + (t_1 - t_repeated) / G + t_comm(G), with
      CAConv, n_in < G (ResNet-20): Slide_f is repeated on every rank (n_in (f^2 - 1) hoisted rotations at the
        measured hoisted rate); outputs all-gathered;
      CAConv, n_in >= G (ResNet-18): Slide sharded by input; slid ciphertexts and outputs all-gathered;
      RAConv, n_o < G (ResNet-20): taps sharded; one all-reduce of the lazy-sum state, then the ModDown, rescale,
        RaS_g / IR_g repeated on every rank (their plain rotations at the measured plain rate);
      RAConv, n_o >= G: outputs sharded and all-gathered.
    Transfers at NVLINK_GBS per direction; all-gather moves (G-1)/G of the data into each rank."""
    N_ = N
    ct_in = 2 * (level + 1) * N_ * 8
    ct_out = 2 * (p.out_level(level) + 1) * N_ * 8
    f2 = p.f * p.f
    out = {}
    for G in (2, 4, 8):
        frac = (G - 1) / G
        if algo == "CA":
            if p.n_in >= G:
                rep = 0.0
                comm = frac * (p.n_in * f2 * ct_in + p.n_out * ct_out) / (NVLINK_GBS * 1e9) * 1e3
            else:
                rep = 1e3 * p.n_in * (f2 - 1) / hoisted_rate if f2 > 1 else 0.0
                comm = frac * p.n_out * ct_out / (NVLINK_GBS * 1e9) * 1e3
        else:
            if p.n_out < G:
                tail = p.counts["RaS_g"] + p.counts["IR_g"]
                rep = 1e3 * (p.n_out + tail) / plain_rate
                state = (2 * (level + 1 + 4) + 2 * (level + 1)) * N_ * 8 * p.n_out
                comm = 2 * frac * state / (NVLINK_GBS * 1e9) * 1e3
            else:
                rep = 0.0
                comm = frac * p.n_out * ct_out / (NVLINK_GBS * 1e9) * 1e3
        rep = min(rep, ms)
        tg = rep + (ms - rep) / G + comm
        out[f"G{G}"] = {"ms": tg, "speedup": ms / tg, "repeated_ms": rep, "comm_ms": comm}
    return out


def layer_roofline(p, algo: str, level: int, ms: float, kp: int = 4, alpha: int = 4):
    """Per-layer roofline fractions: HBM -- algorithmic bytes (input cts, the stored weight
    plaintexts and mask, one read of every distinct evaluation-key slice the layer uses, output cts; intermediates
    excluded) over the layer time vs MEASURED_PEAKS hbm_gbs; FP64 -- the layer's key switches by variant (CAConv
    Slide: hoisted groups, RAConv Slide: lazy HRotSum, RaS / RaS_g / IR_g: plain) + PMult terms + rescales, in
    FP64-pipe ops, vs 148 x 64 x 1.965 GHz."""
    pk = peaks()
    n = level + 1
    out_level = p.out_level(level)
    beta = (n + alpha - 1) // alpha
    ct = lambda lv: 2 * (lv + 1) * N * 8  # noqa: E731
    key_slice = 2 * beta * (n + kp) * N * 6
    alg = p.n_in * ct(level) + p.n_pt * n * N * 8 + (level * N * 8 if p.has_mask else 0) + \
        len(p.rots) * key_slice + p.n_out * ct(out_level)
    c = p.counts
    lv2 = level - 1  # RaS / RaS_g / IR_g run after the SISO rescale
    ops = 0.0
    if algo == "CA":
        if c["Slide"]:
            ops += p.n_in * ks_fp64_ops(level, "modup") + c["Slide"] * ks_fp64_ops(level, "hoisted")
    else:
        ops += c["Slide"] * ks_fp64_ops(level, "lazy_term") + p.n_out * ks_fp64_ops(level, "moddown")
    ops += (c["RaS"] + c["RaS_g"] + c["IR_g"]) * ks_fp64_ops(lv2, "plain")
    ops += c["PMult"] * 2 * n * N * 7
    resc = 2 * (2 * 8 * (N // 2) * 8 * 2) + 2 * n * (2 * 8 * (N // 2) * 8)  # per rescale: 2 iNTT + 2l NTT limbs
    ops += (p.n_out + (p.n_out if p.has_mask else 0)) * resc
    t = ms * 1e-3
    fp64_peak = 148 * 64 * 1.965e9
    return {"alg_bytes": alg, "hbm_gbs": alg / t / 1e9, "hbm_frac": alg / t / 1e9 / pk["hbm_gbs"],
            "fp64_ops": ops, "fp64_tops": ops / t / 1e12, "fp64_frac": ops / t / fp64_peak,
            "bound": "fp64" if ops / fp64_peak > alg / (pk["hbm_gbs"] * 1e9) else "hbm"}


def keyset_report(log_n: int = 16):
    """f2 (tb:Rot and Boot P:1147-1168): the networks' conv rotations under limited
    rotation-key sets (host-side plans; DESIGN R-KEYSET).  Readings of the loaded set: every key the plans need;
    the Slide keys + both-sign powers of two (bootstrapping's power-of-two rotation keys); the Slide keys + positive
    powers of two only; the Slide keys only.  Reported: loaded keys, their memory (6-byte packed and at the paper's
    168 MB), conv rotations and "eff. total" (each synthesized rotation counted once per key switch)."""
    import paper_2302_02407_b200 as hy
    n = 1 << (log_n - 1)
    pow2 = [1 << i for i in range(log_n - 1)]
    key_mib = 2 * 6 * 28 * (1 << log_n) * 6 / 2**20
    out = {}
    for net, layers in (("ResNet-20", R20_LAYERS), ("ResNet-18", R18_LAYERS)):
        plans = []
        slide = set()
        for name, spec, mult in layers:
            S = spec[10] if len(spec) > 10 else 1
            plans.append((name, hy.ConvPlan(None, *spec[:10], log_n=log_n, S=S), mult))
            slide |= {t % n for t in _tap_amounts(spec) if t % n}
        slide = sorted(slide)
        rows = {}
        for kname, extra in (("all_needed", None), ("slide+pm2i", pow2 + [n - x for x in pow2]),
                             ("slide+p2i", pow2), ("slide_only", [])):
            ks = None if extra is None else hy.KeySet(log_n, slide + extra)
            tot = eff = 0
            used = set()
            for name, p, mult in plans:
                p.set_keyset(ks)
                c, e = p.counts, p.eff_counts
                tot += mult * sum(c[k] for k in ("Slide", "RaS", "RaS_g", "IR_g"))
                eff += mult * sum(e[k] for k in ("Slide", "RaS", "RaS_g", "IR_g"))
                used |= set(p.rots)
            nk = len(used)
            rows[kname] = {"loaded_keys_used": nk, "conv_rotations": tot, "eff_total": eff,
                           "evk_gib_packed": nk * key_mib / 1024, "evk_gib_8byte_words": nk * 168 / 1024}
        out[net] = rows
    out["paper"] = {"ResNet-20": {"total": 919, "eff_total": 1002}, "ResNet-18": {"total": 7359, "eff_total": 9095},
                    "evks": "66 unique Evks = 11.1 GB at Set_hyp (P:1243); one Evk = 2 x 6 x 28 limbs x 512 KiB = "
                            "168 MiB (P:1208), i.e. 176 MB (P:1240), and 66 x 168 MiB = 11.1 GiB",
                    "note": "the paper's totals include its IR layout (lost figures, P:996-1000); ours count the "
                            "plans of DESIGN R-LAYOUT / R-DSCONV (stem excluded for ResNet-18)"}
    return out


def plan_search_report():
    """f3: the (m, d) plan search of paper_2302_02407_b200.planner over the product's
    implementable plans, ranked by the paper's per-operation CPU costs (tb:Benchmark P:148); host only."""
    from paper_2302_02407_b200 import planner as P
    out = {}
    for net in (P.RESNET20, P.RESNET18):
        out[net.name] = [{"mds": p.fmts, "conv_rotations": p.rotations, "pmults": p.pmults, "boots": p.boots,
                          "modelled_cpu_s": p.time_ms() / 1000} for p in P.search(net)]
    out["paper_optimal"] = {"ResNet-20": {"mds": [[1, 2], [2, 4], [4, 8]], "boots": 10, "cpu_s": 37.57},
                            "ResNet-18": {"mds": [[1, 1], [2, 2], [4, 4], [8, 8]], "boots": 65, "cpu_s": 356.97}}
    return out


def _tap_amounts(spec):
    ci, co, w, f, s, wp, g = spec[:7]
    pad = (f - 1) // 2
    return [(j1 - pad) * g * wp + (j2 - pad) * g for j1 in range(f) for j2 in range(f)]


def bench_conv(ctx, ws, rank, steps, warmup, timed, layers_def=None, net="ResNet-20", rates=(41000.0, 30000.0)):
    """Per-layer device time of every conv layer type (fresh encryption at its scheduled level,
    outputs sharded over ranks + all-gathered), and the network's conv total.  rates: measured hoisted (l+1 = 10)
    and plain (l+1 = 7) keyswitch/s for the scaling model."""
    import torch

    import paper_2302_02407_b200 as hy
    from paper_2302_02407_b200.dist import all_gather_cts, caconv_slide_sharded, raconv_tap_sharded, shard

    sk, ek = synth.SEED_SK, synth.SEED_EVK
    keys = {}
    layers = {}
    total = 0.0
    for li, (name, spec, mult) in enumerate(layers_def or R20_LAYERS):
        ci, co, w, f, s, wp, g, m, d, algo = spec[:10]
        S = spec[10] if len(spec) > 10 else 1
        p = hy.ConvPlan(ctx, ci, co, w, f, s, wp, g, m, d, algo, S=S)
        level = CA_LEVEL if algo == "CA" else RA_LEVEL
        for r in p.rots:
            if r not in keys:
                keys[r] = ctx.keygen_rot(sk, ek, r)
        K = synth.conv_weight(2000 + li, co, ci, f)
        pts = p.encode_weights(K, level)
        scale = 2 ** synth.PARAMS["hyp"]["log_scale"]
        cts = [ctx.encrypt(sk, synth.SEED_ENC, 10_000 + 100 * li + i,
                           ctx.encode(synth.slots_uniform(3000 + 100 * li + i, ctx.n), scale, level), level)
               for i in range(p.n_in)]
        b, e = shard(p.n_out, rank, ws)
        lo = p.out_level(level)
        outs = [ctx.empty(*ctx.ct_shape(lo)) for _ in range(e - b)]
        scratch = p.scratch(level)
        like = ctx.empty(*ctx.ct_shape(lo))
        evks = [keys[r] for r in p.rots]

        tap_shard = algo == "RA" and ws > 1 and p.n_out < ws  # ResNet-20 RAConv: one output, shard the taps
        # CAConv with at least one input per rank (ResNet-18): shard Slide_f by input and all-gather the slid
        # ciphertexts instead of repeating every Slide rotation on every rank
        slide_shard = algo == "CA" and ws > 1 and p.n_in >= ws and f > 1  # pconv (f = 1) has no Slide

        def step():
            if tap_shard:  # every rank ends with every output: no gather
                return [raconv_tap_sharded(p, evks, cts, level, pts, o, scratch) for o in range(p.n_out)]
            if slide_shard:
                return caconv_slide_sharded(p, evks, cts, level, pts, scratch)
            if e > b:
                p.run(evks, cts, level, pts, scratch, b, e, outs)
            if ws > 1:
                return all_gather_cts(outs, p.n_out, like)
            return outs

        ms, launches = timed(step, steps, warmup)
        identity = None
        if ws > 1:
            # the sharded, combined result equals a single-rank run bit for bit -- rank 0
            # recomputes the last output (owned by the last rank, or tap-sharded) alone and compares its limbs
            got = step()
            j = p.n_out - 1
            if rank == 0:
                alone = p.run(evks, cts, level, pts, scratch, j, j + 1)[0]
                identity = {"output": j, "bit_identical": bool(torch.equal(got[j], alone)),
                            "how": "rank 0 recomputes the output alone and compares every limb"}
            barrier(ws)
        # one extra instrumented run: device ms per kernel family (CUDA events on the launching stream)
        ctx.time_kernels(sum(ctx.FAMILIES.values()))
        step()
        torch.cuda.synchronize()
        fams = {}
        for fn, fm in ctx.FAMILIES.items():
            t, n, _ = ctx.kernel_times(fm)
            if n:
                fams[fn] = round(t, 3)
        ctx.time_kernels(0)
        layers[name] = {"ms": ms, "mult": mult, "n_in": p.n_in, "n_out": p.n_out, "level_in": level,
                        "roofline": layer_roofline(p, algo, level, ms),
                        "scaling_model": scaling_model(p, algo, level, ms, rates[0], rates[1]) if ws == 1 else None,
                        "sharding": "taps (all-reduce)" if tap_shard else (
                            "Slide by input + outputs (two all-gathers)" if slide_shard else (
                                "outputs (all-gather)" if ws > 1 else None)),
                        "rotations": p.counts, "gpu_launches": launches, "weight_pts": p.n_pt, "prcr_segments": S,
                        "multi_gpu_check": identity,
                        "family_ms": fams}
        total += mult * ms
        del pts, cts, outs, scratch
        torch.cuda.empty_cache()
    if net == "ResNet-20":
        note = ("sum over the 19 3x3 convs + 2 pconv of per-layer device time (max over ranks), each layer on a "
                "fresh encryption at its scheduled level; bootstrapping/activation excluded (P:1095-1101 conv "
                "columns: 0.52 s on A100, context only)")
    else:
        note = ("sum over the 19 convs after the stem (13 stride-1 3x3 convs with PRCR |S|=8, 3 stride-2 dsconv and "
                "3 pconv shortcuts with full weights) of per-layer device time, each layer on a fresh encryption at "
                "its scheduled level; context: ResNet-18 conv 7.59 s on A100 (P:1095-1096)")
    # the evaluation keys the network's conv layers use (every non-Slide amount is +-2^i, i.e. in a bootstrapping
    # key set, so no rotation has to be decomposed into loaded keys; P:1242-1245 loads 66 keys for ResNet-18)
    n_keys = len(keys)
    key_info = {"distinct_rotation_keys": n_keys, "gib_at_full_level": n_keys * ctx.evk_bytes() / 2**30,
                "non_slide_amounts_all_power_of_two": True}
    model = None
    if ws == 1:
        model = {}
        for G in (2, 4, 8):
            tg = sum(v["mult"] * v["scaling_model"][f"G{G}"]["ms"] for v in layers.values())
            model[f"G{G}"] = {"total_ms": tg, "speedup": total / tg}
    return {"layers": layers, "total_ms": total, "n_gpus": ws, "network": net, "note": note, "keys": key_info,
            "scaling_model": model}


def bench_blocks(ctx, ws, rank, steps, warmup, timed):
    """ResNet-20 basic-block conv halves (Alg. 3): stride-1 CAConv -> x^2 (MulCt + relinearization
    + rescale) -> RAConv, device-timed as one step per stage (CAConv input at l+1 = 10).  Every rank
    runs the whole block (weak scaling is the HRot microbenchmark's; the layer tables shard)."""
    import torch

    import paper_2302_02407_b200 as hy

    sk, ek = synth.SEED_SK, synth.SEED_EVK
    rlk = ctx.keygen_relin(sk, ek)
    scale = 2 ** synth.PARAMS["hyp"]["log_scale"]
    spec = {name: sp for name, sp, _ in R20_LAYERS}
    out = {}
    for stage, (ca_n, ra_n) in enumerate([("L1_ca", "L1_ra"), ("L2_ca", "L2_ra"), ("L3_ca", "L3_ra")]):
        plans = []
        for nm in (ca_n, ra_n):
            ci, co, w, f, s_, wp, g, m, d, algo = spec[nm][:10]
            plans.append(hy.ConvPlan(ctx, ci, co, w, f, s_, wp, g, m, d, algo))
        blk = hy.ConvBlock(ctx, *plans)
        mid, ra_level, out_level = blk.levels(CA_LEVEL)
        keys = [{r: ctx.keygen_rot(sk, ek, r) for r in p.rots} for p in plans]
        K1 = synth.conv_weight(5000 + stage, spec[ca_n][1], spec[ca_n][0], 3)
        K2 = synth.conv_weight(5100 + stage, spec[ra_n][1], spec[ra_n][0], 3)
        pts = [plans[0].encode_weights(K1, CA_LEVEL), plans[1].encode_weights(K2, ra_level)]
        cts = [ctx.encrypt(sk, synth.SEED_ENC, 20_000 + 100 * stage + i,
                           ctx.encode(synth.slots_uniform(6000 + 100 * stage + i, ctx.n), scale, CA_LEVEL), CA_LEVEL)
               for i in range(plans[0].n_in)]
        scr = [plans[0].scratch(CA_LEVEL), plans[1].scratch(ra_level)]

        def step():
            blk.run(keys[0], keys[1], rlk, cts, CA_LEVEL, pts[0], pts[1], scr[0], scr[1])

        ms, launches = timed(step, steps, warmup)
        mids = [ctx.empty(*ctx.ct_shape(mid)) for _ in range(plans[0].n_out)]

        def sq_step():
            x = ctx.square_batch(rlk, mids, mid, outs=mids)
            for c in x:
                ctx.rescale(c, mid)

        ms_sq, _ = timed(sq_step, steps, warmup)
        out[f"stage{stage + 1}"] = {"ms": ms, "square_ms": ms_sq, "ca": ca_n, "ra": ra_n, "level_in": CA_LEVEL,
                                    "level_ra": ra_level, "level_out": out_level, "n_square": plans[0].n_out,
                                    "gpu_launches": launches}
        del pts, cts, scr, keys, mids
        torch.cuda.empty_cache()
    return {"blocks": out, "note": "CAConv -> x^2 -> RAConv per stage (Alg. 3, P:739-765), device time; the "
                                   "square is MulCt + relinearization + rescale of the n_o CAConv outputs"}


# --------------------------------------------------------------------------- C1 (BASELINE configs[0])
C1_SPEC = (4, 4, 8, 3, 1, 8, 1, 1, 1, "RA")  # single 3x3 RAConv 4->4, 8x8, N=2^12


def bench_c1(device, steps, warmup, timed_fn, with_oracle=True):
    """BASELINE configs[0]: one 3x3 RAConv 4 -> 4 channels on an 8x8 image, N = 2^12, 3 RNS limbs + 1 special
    prime (toy set), inputs encrypted at l = 2: device time per layer call, and the CPU oracle's time for the same
    layer (full oracle, all outputs) on the host cores."""
    import torch

    import paper_2302_02407_b200 as hy
    prm = synth.PARAMS["toy"]
    ctx = hy.Context(**prm, device=device)
    sk, ek = synth.SEED_SK, synth.SEED_EVK
    p = hy.ConvPlan(ctx, *C1_SPEC)
    level = len(prm["q_bits"]) - 1
    X = synth.image(1, 4, 8)
    K = synth.conv_weight(2, 4, 4, 3)
    scale = 2 ** prm["log_scale"]
    # the layer's work is data-independent: seeded uniform slots stand in for the packed image on the GPU leg
    cts = [ctx.encrypt(sk, 900, i, ctx.encode(synth.slots_uniform(40 + i, ctx.n), scale, level), level)
           for i in range(p.n_in)]
    evks = [ctx.keygen_rot(sk, ek, r) for r in p.rots]
    pts = p.encode_weights(K, level)
    scratch = p.scratch(level)
    outs = [ctx.empty(*ctx.ct_shape(p.out_level(level)))]
    ms, _ = timed_fn(lambda: p.run(evks, cts, level, pts, scratch, 0, 1, outs), steps, warmup)
    torch.cuda.synchronize()
    l0 = ctx.launch_count()  # this context's kernels per layer call (timed_fn counts the bench context's)
    p.run(evks, cts, level, pts, scratch, 0, 1, outs)
    launches = ctx.launch_count() - l0
    res = {"workload": "C1: 3x3 RAConv 4->4, 8x8, N=2^12, 3 limbs + 1 special prime, l = 2 (BASELINE configs[0])",
           "ms": ms, "gpu_launches": launches, "rotations": p.counts, "n_in": p.n_in, "n_out": p.n_out}
    if with_oracle:  # the cpu_baseline leg: the oracle's encrypted execution of the same layer
        import oracle
        from oracle import hyphen as H
        o = oracle.Oracle(**prm)
        plan = H.plan_raconv(H.ConvSpec(*C1_SPEC, n=o.n), K)
        octs = [o.encrypt(sk, 900, i, o.encode(v, scale, level)) for i, v in enumerate(H.pack(X, plan.fin))]
        oevks = {r: o.keygen_rot(sk, ek, r) for r in H.rotation_amounts(plan, o.n)}
        enc = H.EncConv(o, plan, oevks)
        enc.run(octs)  # warm (weight encoding cache)
        t0 = time.perf_counter()
        n_rep = 3
        for _ in range(n_rep):
            enc.run(octs)
        res["oracle_ms"] = 1000.0 * (time.perf_counter() - t0) / n_rep
        res["oracle_cores"] = os.cpu_count()
        res["oracle_over_gpu"] = res["oracle_ms"] / ms
    del ctx
    return res


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_rate_threads(n_rot: int, threads: int):
    """oracle_keyswitch_rate in a fresh process with OMP_NUM_THREADS = threads (the C oracle's OpenMP pool is
    sized when the library loads)."""
    env = dict(os.environ, OMP_NUM_THREADS=str(threads))
    code = ("import json, bench; r, dt = bench.oracle_keyswitch_rate(%d); print(json.dumps([r, dt]))" % n_rot)
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True,
                         timeout=900)
    r, dt = json.loads(out.stdout.strip().splitlines()[-1])
    return r, dt


def bench_boot_linear(ctx, steps, warmup, timed):
    """The bootstrapping linear steps (partial; DESIGN R-LINTRANS) at Set_hyp: ModRaise of a
    level-0 ciphertext to level 23, and one BSGS diagonal linear transform at level 23 with 32 diagonals (a radix-32
    CoeffToSlot layer's shape: d = 0..31 x stride 1, baby-step size 8: 7 hoisted baby rotations, 3 giant rotations in
    one lazy HRotSum, 32 PMults, one rescale).  Device time per call; random diagonals (the work is data-independent)."""
    import numpy as np

    import paper_2302_02407_b200 as hy
    sk, ek = synth.SEED_SK, synth.SEED_EVK
    lv = LEVEL
    scale = 2 ** synth.PARAMS["hyp"]["log_scale"]
    ct = ctx.encrypt(sk, synth.SEED_ENC, 77, ctx.encode(synth.slots_uniform(77, ctx.n), scale, lv), lv)
    ct0 = ctx.level_down(ct, lv, 0)
    raised = ctx.empty(*ctx.ct_shape(lv))
    ms_raise, l_raise = timed(lambda: ctx.mod_raise(ct0, lv, raised), steps, warmup)
    ds = list(range(32))
    lt = hy.LinTrans(ctx, ds, 8)
    keys = {r: ctx.keygen_rot(sk, ek, r) for r in lt.rots}
    g = np.random.default_rng(5)
    pts = lt.encode([g.uniform(-1, 1, ctx.n) + 1j * g.uniform(-1, 1, ctx.n) for _ in ds], lv)
    out = ctx.empty(*ctx.ct_shape(lv - 1))
    scratch = ctx.empty(int(hy.lib().hy_lintrans_scratch_words(ctx._c, lt._p, lv)))
    ms_lt, l_lt = timed(lambda: lt.apply(keys, raised, lv, pts, scratch, out), steps, warmup)
    small = bench_bootstrap_small(steps, warmup, timed)
    del keys, pts, raised, out, scratch
    hyp = bench_bootstrap_set_hyp(ctx, steps)
    chain = hyp.pop("chain", None)
    return {"mod_raise_ms": ms_raise, "mod_raise_launches": l_raise, "lintrans_ms": ms_lt, "lintrans_launches": l_lt,
            "bootstrap_n1024": small, "bootstrap_set_hyp": hyp, "resnet20_chain": chain,
            "lintrans": {"diagonals": len(ds), "baby_steps": lt.n_baby, "giant_steps": lt.n_giant, "level": lv,
                         "keys": len(lt.rots)},
            "note": "Set_hyp: ModRaise + one BSGS diagonal transform (the CoeffToSlot / SlotToCoeff building block); "
                    "the whole bootstrapping at Set_hyp with factorised transforms (bootstrap_set_hyp, DESIGN R-SFFT) "
                    "and at N = 2^10 with dense ones (bootstrap_n1024)"}


def bench_bootstrap_set_hyp(ctx, steps):
    """The whole bootstrapping at Set_hyp (N = 2^16, L+1 = 24, h = 192; DESIGN R-SFFT,
    R-EVALMOD): ModRaise 0 -> 23, CoeffToSlot as 3 factorised levels (63/63/32 diagonals), EvalMod (degree-30
    Chebyshev series of cos(12 s), 4 double angles), SlotToCoeff as 3 levels -> level 6 (L' = 6).  Device
    time per call with every key and transform plaintext resident (encoded once, untimed, like weights), set beside
    the paper's Boot = 2160 ms (tb:Benchmark; HEaaN, its own hardware: context, not a target)."""
    import math

    import numpy as np
    import torch

    from paper_2302_02407_b200.boot import Bootstrapper, level_bs, sfft_levels, transform_rots
    sk, ek = synth.SEED_SK, synth.SEED_EVK
    N, top = ctx.N, ctx.n_q - 1
    r, a = 4, 12.0
    K = float(ctx.moduli[0]) / 2**42
    cts = sfft_levels(N, [5, 5, 5], inverse=True, scale=0.5)
    stc = sfft_levels(N, [5, 5, 5], scale=K / (2 * math.pi))
    bs = ([level_bs(D) for D in cts], [level_bs(D) for D in stc])
    rots = sorted(set(transform_rots(ctx, cts, bs[0])) | set(transform_rots(ctx, stc, bs[1])))
    keys = {rr: ctx.keygen_rot(sk, ek, rr) for rr in rots}
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda x: np.cos(a * x), 30)
    cheb[1::2] = 0.0
    bt = Bootstrapper(ctx, cts, stc, bs, cheb, r, a, keys, ctx.keygen_galois(sk, ek, 2 * N - 1),
                      ctx.keygen_relin(sk, ek))
    z = synth.slots_uniform(6, ctx.n)
    ct = ctx.encrypt(sk, synth.SEED_ENC, 6, ctx.encode(z, 2**42, top), top)
    ct0 = ctx.level_down(ct, top, 0)
    out = bt.bootstrap(ct0, 2.0**42, top)  # encodes the transform plaintexts once (untimed)
    out = bt.bootstrap(ct0, 2.0**42, top)  # and once more: the caching allocator reaches its steady state
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_it = max(1, min(steps, 3))
    l0 = ctx.launch_count()
    e0.record()
    for _ in range(n_it):
        out = bt.bootstrap(ct0, 2.0**42, top)
    e1.record()
    torch.cuda.synchronize()
    got = ctx.decode(ctx.decrypt(sk, out.t, out.level), out.level, out.scale)
    err = float(np.max(np.abs(got - z)) / np.max(np.abs(z)))
    ms, launches = e0.elapsed_time(e1) / n_it, (ctx.launch_count() - l0) // n_it
    graph = {}
    try:  # the same sequence captured once in a CUDA graph and replayed (no host sequencing in the timed region)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            bt.bootstrap(ct0, 2.0**42, top)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            gout = bt.bootstrap(ct0, 2.0**42, top)
        g.replay()
        torch.cuda.synchronize()
        ok = bool(torch.equal(gout.t, out.t))
        e0.record()
        for _ in range(n_it):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph = {"ms": e0.elapsed_time(e1) / n_it, "replay_equals_eager": ok}
        del g, gout
    except Exception as ex:  # noqa: BLE001 -- reported, not fatal
        graph = {"error": str(ex)[:200]}
    res = {"ms": ms, "calls": n_it, "launches": launches, "cuda_graph": graph,
            "levels": [top, out.level], "levels_consumed": top - out.level, "rotation_keys": len(rots),
            "transform_levels": {"coeff_to_slot": [len(D) for D in cts], "slot_to_coeff": [len(D) for D in stc]},
            "evalmod": {"cos_a": a, "double_angles": r, "chebyshev_degree": 30},
            "max_rel_error": err, "paper_boot_ms": 2160.0,
            "note": "host-sequenced C-ABI calls on the resident keys; the paper's 2160 ms is HEaaN on its own "
                    "hardware (tb:Benchmark), context only"}
    res["chain"] = bench_block_chain(ctx, bt, sk, ek)
    return res


R20_BLOCKS = [  # the three stages' regular blocks (ResNet-20 CIFAR-10): CAConv, x^2, RAConv + shortcut
    ("stage1", (16, 16, 32, 3, 1, 32, 1, 1, 2, "CA"), (16, 16, 32, 3, 1, 32, 1, 2, 1, "RA"), 3),
    ("stage2", (32, 32, 16, 3, 1, 32, 2, 2, 4, "CA"), (32, 32, 16, 3, 1, 32, 2, 4, 2, "RA"), 3),
    ("stage3", (64, 64, 8, 3, 1, 32, 4, 4, 8, "CA"), (64, 64, 8, 3, 1, 32, 4, 8, 4, "RA"), 3),
]


def bench_block_chain(ctx, bt, sk, ek):
    """Conv blocks chained through Set_hyp bootstrapping (paper_2302_02407_b200.boot.BlockChain):
    per stage of ResNet-20, y = RAConv(CAConv(x)^2) + x at L' = 6 and the refresh (scale set, bootstrap) back to L',
    device-timed per call on random Kaiming weights; tests/test_gpu_boot.py::test_block_chain_set_hyp checks the
    decryption against the plaintext recursion."""
    import numpy as np
    import torch

    import paper_2302_02407_b200 as hy
    from paper_2302_02407_b200.boot import CT, BlockChain
    L = 6
    chain = BlockChain(ctx, bt)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    out = {}
    for name, cs, rs, count in R20_BLOCKS:
        ca, ra = hy.ConvPlan(ctx, *cs), hy.ConvPlan(ctx, *rs)
        blk = hy.ConvBlock(ctx, ca, ra)
        _, ra_level, out_level = blk.levels(L)
        cak = {r: ctx.keygen_rot(sk, ek, r) for r in ca.rots}
        rak = {r: ctx.keygen_rot(sk, ek, r) for r in ra.rots}
        cap = ca.encode_weights(synth.conv_weight(5, cs[1], cs[0], 3) * 0.3, L)
        rap = ra.encode_weights(synth.conv_weight(6, rs[1], rs[0], 3) * 0.3, ra_level)
        x0 = CT(ctx.encrypt(sk, 7, 0, ctx.encode(synth.slots_uniform(7, ctx.n), 2**42, L), L), L, 2.0**42)
        y = chain.block(blk, cak, rak, cap, rap, x0)
        z = chain.refresh(y)  # warm-up (encodes the refresh constants)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            y = chain.block(blk, cak, rak, cap, rap, x0)
        e1.record()
        torch.cuda.synchronize()
        ms_b = e0.elapsed_time(e1) / 3
        e0.record()
        for _ in range(3):
            z = chain.refresh(y)
        e1.record()
        torch.cuda.synchronize()
        ms_r = e0.elapsed_time(e1) / 3
        out[name] = {"block_ms": ms_b, "refresh_ms": ms_r, "blocks_in_resnet20": count, "levels": [L, out_level, z.level]}
        del cak, rak, cap, rap
    # the whole ResNet-20 conv stack end to end (boot.ResNet20Convs): stem, 9 blocks, 8 bootstraps
    from paper_2302_02407_b200.boot import ResNet20Convs
    shapes = [((16, 3), 3)] + [((16, 16), 3)] * 6 + [((32, 16), 3), ((32, 32), 3), ((32, 16), 1)] + \
        [((32, 32), 3)] * 4 + [((64, 32), 3), ((64, 64), 3), ((64, 32), 1)] + [((64, 64), 3)] * 4
    net = ResNet20Convs(ctx, chain, [synth.conv_weight(200 + i, co, ci, f) * 0.5 for i, ((co, ci), f) in
                                     enumerate(shapes)], lambda r: ctx.keygen_rot(sk, ek, r))
    Li = net.input_level
    x = CT(ctx.encrypt(sk, 32, 0, ctx.encode(synth.slots_uniform(8, ctx.n), 2**42, Li), Li), Li, 2.0**42)
    y = net.run(x)  # warm-up
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    e0.record()
    for _ in range(2):
        y = net.run(x)
    e1.record()
    torch.cuda.synchronize()
    ms_e = e0.elapsed_time(e1) / 2
    launches = (ctx.launch_count() - l0) // 2
    graph = {}
    try:  # the whole network captured once in a CUDA graph and replayed (no host sequencing in the timed region)
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            net.run(x)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            gy = net.run(x)
        g.replay()
        torch.cuda.synchronize()
        ok = bool(torch.equal(gy.t, y.t))
        e0.record()
        for _ in range(2):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        graph = {"ms": e0.elapsed_time(e1) / 2, "replay_equals_eager": ok}
        del g, gy
    except Exception as ex:  # noqa: BLE001 -- reported, not fatal
        graph = {"error": str(ex)[:200]}
    e2e = {"ms": ms_e, "cuda_graph": graph, "launches": launches, "bootstraps": 8,
           "convs": 21 + 3, "input_level": Li, "output_level": y.level, "paper_a100_s": 1.40,
           "note": "stem conv + square, 9 blocks y = RAConv(CAConv(x)^2) + s(x) (dsconv / pconv at the stage "
                   "boundaries; 1x1 identity RAConvs convert the stem's and the pconvs' RA format), a bootstrap after "
                   "each of the first 8 blocks; no pooling / FC; random Kaiming weights x 0.5; "
                   "tests/test_gpu_boot.py::test_resnet20_convs_end_to_end checks the decryption against the "
                   "plaintext network (8.9e-4 of its max, r02v)"}
    return {"stages": out, "level_in": L, "resnet20_end_to_end": e2e,
            "note": "y = RAConv(CAConv(x)^2) + x, then bootstrap (BlockChain.refresh) back to L' = 6; device time per "
                    "call, host-sequenced C-ABI calls"}


def bench_bootstrap_small(steps, warmup, timed):
    """The whole bootstrapping (DESIGN R-EVALMOD) on the 'boot' chain (N = 2^10, 17 limbs), device time per call
    with every key resident; timed through the bench's own context clock (the launches are this context's)."""
    import math

    import numpy as np
    import torch

    import paper_2302_02407_b200 as hy
    from paper_2302_02407_b200.boot import Bootstrapper
    prm = synth.PARAMS["boot"]
    ctx = hy.Context(**prm, device=torch.cuda.current_device())
    sk, ek = synth.SEED_SK, synth.SEED_EVK
    n, N, top = ctx.n, ctx.N, len(prm["q_bits"]) - 1
    r, a, bs = 3, 8.0, 32
    K = float(ctx.moduli[0]) / 2**40
    # the special-FFT matrix V[j][k] = zeta^{k 5^j} (DESIGN R-LINTRANS) and its diagonals
    rot = np.array([pow(5, j, 2 * N) for j in range(n)], dtype=np.int64)
    V = np.exp(1j * np.pi * (np.outer(rot, np.arange(n)) % (2 * N)) / N)
    j = np.arange(n)
    diag = lambda M: [M[j, (j + d) % n] for d in range(n)]  # noqa: E731
    cheb = np.polynomial.chebyshev.chebinterpolate(lambda x: np.cos(a * x), 30)
    cheb[1::2] = 0.0
    lt = hy.LinTrans(ctx, list(range(n)), bs)
    keys = {rr: ctx.keygen_rot(sk, ek, rr) for rr in lt.rots}
    bt = Bootstrapper(ctx, diag(np.linalg.inv(V) / 2), diag(K / (2 * math.pi) * V), bs, cheb, r, a, keys,
                      ctx.keygen_galois(sk, ek, 2 * N - 1), ctx.keygen_relin(sk, ek))
    ct = ctx.encrypt(sk, synth.SEED_ENC, 5, ctx.encode(synth.slots_uniform(5, n), 2**40, top), top)
    ct0 = ctx.level_down(ct, top, 0)
    bt.bootstrap(ct0, 2.0**40, top)  # encodes the transform plaintexts once (untimed, like weights)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launch_count()
    e0.record()
    for _ in range(steps):
        out = bt.bootstrap(ct0, 2.0**40, top)
    e1.record()
    torch.cuda.synchronize()
    res = {"ms": e0.elapsed_time(e1) / steps, "launches": (ctx.launch_count() - l0) // steps, "levels_consumed":
           top - out.level, "ring": "N = 2^10, 17 limbs (synth boot chain)",
           "note": "host-sequenced C-ABI calls; the transforms are dense (512 diagonals each)"}
    # the same sequence captured once in a CUDA graph and replayed (the small ring is launch-bound)
    try:
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            bt.bootstrap(ct0, 2.0**40, top)  # warm the allocator on the capture stream
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            gout = bt.bootstrap(ct0, 2.0**40, top)
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        ok = bool(torch.equal(gout.t, out.t))
        e0.record()
        for _ in range(steps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        res["cuda_graph"] = {"ms": e0.elapsed_time(e1) / steps, "replay_equals_eager": ok}
    except Exception as ex:  # noqa: BLE001 -- reported, not fatal
        res["cuda_graph"] = {"error": str(ex)[:200]}
    return res


# --------------------------------------------------------------------------- our arm
def run_ours(args, ws, rank, local):
    import torch

    import paper_2302_02407_b200 as hy

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    prm = synth.PARAMS["hyp"]
    ctx = hy.Context(**prm, device=local, max_batch=int(os.environ.get("HY_BENCH_BATCH", "64")))  # key switches per launch
    sk, ek = synth.SEED_SK, synth.SEED_EVK
    rs = [i + 1 for i in range(BATCH)]
    # keys (server state) and inputs (client output), resident in HBM before timing
    evks = [ctx.keygen_rot(sk, ek, r) for r in rs]
    scale = 2 ** prm["log_scale"]
    pt = ctx.encode(synth.slots_uniform(1000 + rank, ctx.n), scale, LEVEL)
    cts = [ctx.encrypt(sk, synth.SEED_ENC, rank * BATCH + i, pt, LEVEL) for i in range(BATCH)]
    outs = [ctx.empty(*ctx.ct_shape(LEVEL)) for _ in range(BATCH)]
    houts = [ctx.empty(*ctx.ct_shape(LEVEL)) for _ in range(BATCH)]
    torch.cuda.synchronize()

    stream = torch.cuda.current_stream()

    def step():
        ctx.hrot_batch(evks, cts, LEVEL, rs, outs)

    def step_hoisted():
        ctx.hrot_hoisted(evks, cts[0], LEVEL, rs, houts)

    def timed(fn, k, w):
        for _ in range(w):
            fn()
        torch.cuda.synchronize()
        barrier(ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        l0 = ctx.launch_count()
        prof = os.environ.get("HY_NCU_TIMED") == "1"  # ncu --profile-from-start off captures only this region
        if prof:
            torch.cuda.cudart().cudaProfilerStart()
        e0.record(stream)
        for _ in range(k):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        if prof:
            torch.cuda.cudart().cudaProfilerStop()
        barrier(ws)
        ms = e0.elapsed_time(e1) / k
        return max_over_ranks(ms, ws), (ctx.launch_count() - l0) // k

    with ClockSampler(local) as clk:
        ms, launches = timed(step, args.steps, args.warmup)
    clocks = clk.summary()
    value = BATCH * ws * 1000.0 / ms

    ms_h, _ = timed(step_hoisted, args.steps, max(1, args.warmup // 2))

    # the three HRot variants at the full level and the two conv levels: the same 64 keys
    # and ciphertexts (level l = the first l+1 limbs, a level-down), keyswitch/s and the whole-rotation HBM
    # fraction in algorithmic bytes (ct in once per distinct input, the key slice read, 6-byte packed, ct out)
    variants = None
    if not args.no_variants and os.environ.get("HY_NCU_TIMED") != "1":
        variants = {}
        pk_hbm = peaks()["hbm_gbs"]
        E_ = lambda lv: lv + 1 + len(prm["p_bits"])  # noqa: E731
        for lv in (LEVEL, CA_LEVEL, RA_LEVEL):
            cl = [c[:, : lv + 1].contiguous() for c in cts]
            ol = [ctx.empty(*ctx.ct_shape(lv)) for _ in range(BATCH)]
            o1 = ctx.empty(*ctx.ct_shape(lv))
            ct_b = 2 * (lv + 1) * ctx.N * 8
            key_b = 2 * ctx.n_digits(lv) * E_(lv) * ctx.N * 6
            row = {}
            for vname, fn, moved in (
                    ("plain", lambda: ctx.hrot_batch(evks, cl, lv, rs, ol), BATCH * (2 * ct_b + key_b)),
                    ("hoisted", lambda: ctx.hrot_hoisted(evks, cl[0], lv, rs, ol), ct_b + BATCH * (ct_b + key_b)),
                    ("lazy_sum", lambda: ctx.hrot_sum(evks, cl, lv, rs, o1), BATCH * (ct_b + key_b) + ct_b)):
                t_ms, _ = timed(fn, max(2, args.steps // 2), 2)
                gbs = moved / (t_ms * 1e-3) / 1e9
                row[vname] = {"keyswitch_per_s": BATCH * ws * 1000.0 / t_ms, "ms_per_64": t_ms,
                              "hbm_gbs": gbs, "hbm_frac": gbs / pk_hbm}
            variants[f"l+1={lv + 1}"] = row
            del cl, ol, o1

    # live per-family kernel timing over K instrumented steps (same stream, CUDA events)
    fam = ctx.FAMILIES
    ctx.time_kernels(sum(fam.values()))
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    breakdown = {}
    for name, m in fam.items():
        t, n, by = ctx.kernel_times(m)
        if n:
            breakdown[name] = {"ms_per_step": t / args.steps, "launches_per_step": n // args.steps,
                               "alg_bytes_per_launch": by // n, "avg_us": 1000.0 * t / n}
    ctx.time_kernels(0)
    # the same for the hoisted batch
    ctx.time_kernels(sum(fam.values()))
    for _ in range(args.steps):
        step_hoisted()
    torch.cuda.synchronize()
    breakdown_h = {}
    for name, m in fam.items():
        t, n, by = ctx.kernel_times(m)
        if n:
            breakdown_h[name] = {"ms_per_step": t / args.steps, "launches_per_step": n // args.steps,
                                 "alg_bytes_per_launch": by // n, "avg_us": 1000.0 * t / n}
    ctx.time_kernels(0)
    dominant = max(breakdown, key=lambda k: breakdown[k]["ms_per_step"])
    pk = peaks()
    alpha, kp = 4, 4
    n_l = LEVEL + 1
    E = n_l + kp
    digits = [min(alpha, n_l - j * alpha) for j in range((n_l + alpha - 1) // alpha)]
    # SURVEY 8(d).2 algorithmic bytes of one rotation: ct in + the evaluation-key slice it reads + ct out;
    # intermediates (extended digits, partial sums, conversion rows) excluded.  The key is stored 6 bytes per
    # word; frac_8byte_key_equiv counts it at the paper's 8 bytes per word (168 MB).
    ct_bytes = 2 * n_l * N * 8
    key_slice = 2 * len(digits) * E * N * 6
    key_slice8 = 2 * len(digits) * E * N * 8
    alg_rot = {"plain": (2 * ct_bytes + key_slice, 2 * ct_bytes + key_slice8),
               "hoisted": (ct_bytes + key_slice + ct_bytes / BATCH, ct_bytes + key_slice8 + ct_bytes / BATCH)}

    def ncu_step_bytes(fam_name, bd=None, tfam=None):
        t = ncu_traffic(tfam or fam_name)
        if t is None:
            return None
        # the capture summary holds the per-launch average of the family's kernels
        return t["bytes_per_launch"] * (bd or breakdown)[fam_name]["launches_per_step"]

    def hbm_roof(fam_name, variant="plain", bd=None):
        bd = bd or breakdown
        d = bd[fam_name]
        alg, alg8 = (BATCH * x for x in alg_rot[variant])
        t_s = d["ms_per_step"] * 1e-3
        achieved = alg / t_s / 1e9
        model = d["alg_bytes_per_launch"] * d["launches_per_step"] / t_s / 1e9
        # the hoisted batch's own kernels (tools/ncu_round.py family "<fam>_hoisted") when captured
        tfam = fam_name if variant == "plain" else fam_name + "_hoisted"
        tr = ncu_step_bytes(fam_name, bd, tfam)
        return {"bound": "hbm", "kernel_family": fam_name, "achieved": achieved, "peak": pk["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / pk["hbm_gbs"],
                "frac_8byte_key_equiv": alg8 / t_s / 1e9 / pk["hbm_gbs"],
                "alg_bytes_per_launch": alg / d["launches_per_step"],
                "alg_bytes_def": "SURVEY 8(d).2: (ct in + key slice read + ct out) per rotation x 64 rotations per "
                                 "step, attributed to this family's launches (intermediates excluded)",
                "dram_model_gbs": model,
                "dram_model_note": "the same launches' modelled DRAM bytes including intermediates (extended "
                                   "digits, conversion rows) over their time: achieved DRAM rate, not the roofline",
                **traffic_fields(tfam),
                "traffic_over_alg": None if tr is None else tr / alg,
                "share_of_step": d["ms_per_step"] / ms,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if not pk.get("fallback") else "fallback 6.65 TB/s"}

    fp64_peak = 148 * 64 * 1.965e9 / 1e12  # FP64 lanes x SMs x max clock (B200 unit counts)

    def alu_roof(fam_name, ops_per_launch, what, bd=None):
        d = (bd or breakdown)[fam_name]
        achieved = ops_per_launch / (d["avg_us"] * 1e-6) / 1e12
        tr = ncu_step_bytes(fam_name) if bd is None else None
        return {"bound": "alu", "kernel_family": fam_name, "achieved": achieved, "peak": fp64_peak,
                "unit": "TFP64op/s", "frac": achieved / fp64_peak, **traffic_fields(fam_name),
                "traffic_over_model": None if tr is None else tr / (d["alg_bytes_per_launch"] * d["launches_per_step"]),
                "share_of_step": d["ms_per_step"] / ms, "work": what,
                "peak_source": "148 SM x 64 FP64 lanes x 1.965 GHz (DESIGN.md section 5); one DFMA/DMUL/DADD = 1 op"}

    # algorithmic FP64-pipe work: an NTT column / row pass = 8 stages x N/2
    # butterflies x 8 ops (fmulmod 6 + add + sub); a fast-BConv output word = alpha fmulmods + alpha-1 adds
    # + one fred (3 ops) = 7 alpha + 2
    pass_ops = 8 * (N // 2) * 8
    modup_item = n_l * pass_ops + sum((E - a) * (pass_ops + N * (7 * a + 2)) for a in digits)
    moddown_item = 2 * (kp * pass_ops + n_l * (pass_ops + N * (7 * kp + 2)))
    roofs = {}
    if "modup" in breakdown:
        items = BATCH // breakdown["modup"]["launches_per_step"]
        roofs["modup"] = alu_roof("modup", items * modup_item,
                                  "fused ModUp columns: (l+1) inverse column passes + per digit (E - alpha) x "
                                  "(BConv word + forward column pass), per item")
    if "moddown" in breakdown:  # the fused ModDown column kernel
        items = BATCH // breakdown["moddown"]["launches_per_step"]
        roofs["moddown"] = alu_roof("moddown", items * moddown_item,
                                    "fused ModDown columns: per poly K inverse column passes + (l+1) x (BConv word "
                                    "+ forward column pass), per item")
    for f in ("ntt_ip", "ip", "aut"):
        if f in breakdown:
            roofs[f] = hbm_roof(f)
    for f in ("ntt_a", "ntt_b"):
        if f in breakdown:
            limbs = breakdown[f]["alg_bytes_per_launch"] / (2 * N * 8)
            roofs[f] = alu_roof(f, limbs * pass_ops, "NTT pass: 8 stages x N/2 butterflies x 8 ops per limb")
    roof = roofs.get(dominant) or hbm_roof(dominant)
    # the hoisted batch's dominant family on the same definitions
    roofs_hoisted = {}
    if "ntt_ip" in breakdown_h:
        roofs_hoisted["ntt_ip"] = hbm_roof("ntt_ip", "hoisted", breakdown_h)
    if "moddown" in breakdown_h:
        items = BATCH // breakdown_h["moddown"]["launches_per_step"]
        roofs_hoisted["moddown"] = alu_roof("moddown", items * moddown_item, "fused ModDown columns", breakdown_h)
    # whole-HRot HBM fraction (the metric's "HBM GB/s vs peak"): the bytes a rotation must move -- input ct,
    # its evaluation key, output ct -- over the measured time per rotation (north_star target >= 60 %)
    hrot_hbm = {}
    for name_, t_ms in (("plain", ms), ("hoisted", ms_h)):
        moved, moved8 = alg_rot[name_]
        gbs = moved * BATCH / (t_ms * 1e-3) / 1e9
        hrot_hbm[name_] = {"alg_bytes_per_rotation": moved, "achieved": gbs, "peak": pk["hbm_gbs"], "unit": "GB/s",
                           "frac": gbs / pk["hbm_gbs"],
                           "frac_8byte_key_equiv": moved8 * BATCH / (t_ms * 1e-3) / 1e9 / pk["hbm_gbs"]}
    hrot_hbm["note"] = ("plain: ct in + evk (6-byte packed words) + ct out per rotation; hoisted: the shared input is "
                        "read once per batch, so evk + ct out; frac_8byte_key_equiv counts the key at 8 bytes per "
                        "word (the paper's 168 MB key); the FP64-pipe NTT/BConv work bounds plain HRot below the HBM "
                        "roofline (DESIGN.md section 5)")
    ntt_ms = sum(breakdown[k]["ms_per_step"] for k in ("ntt_a", "ntt_b") if k in breakdown)

    # e2e through the public API with host buffers: pinned H2D of the 64 input cts, D2H of the outputs
    e2e = None
    if not args.no_e2e:
        # chunks of E2E_CHUNK rotations: the H2D of chunk k+1 and the D2H of chunk k-1 run on their own streams
        # while chunk k is key-switched (PCIe is full duplex), so the step costs about one direction's copy time.
        # wire=True: the client holds its ciphertexts in the library's 48-bit wire format (hy_pack48: every
        # residue < 2^48), so 25 % fewer bytes cross PCIe; the device unpacks / packs around the key switches.
        h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream()
        chunks = [(k, min(BATCH, k + E2E_CHUNK)) for k in range(0, BATCH, E2E_CHUNK)]
        dcts = [torch.empty_like(c) for c in cts]

        def make_step(wire):
            if wire:
                hin = [ctx.pack48(c).cpu().pin_memory() for c in cts]
                hout = [torch.empty_like(h).pin_memory() for h in hin]
                din = [torch.empty_like(h, device=dev) for h in hin]
                dout = [torch.empty_like(h, device=dev) for h in hin]
            else:
                hin = [c.cpu().pin_memory() for c in cts]
                hout = [torch.empty_like(c, device="cpu").pin_memory() for c in outs]
                din, dout = dcts, outs

            def e2e_step():
                cur = torch.cuda.current_stream()
                h2d_s.wait_stream(cur)  # the previous step no longer reads the device inputs
                ready = []
                with torch.cuda.stream(h2d_s):
                    for a, b in chunks:
                        for i in range(a, b):
                            din[i].copy_(hin[i], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(h2d_s)
                        ready.append(ev)
                for (a, b), ev in zip(chunks, ready):
                    cur.wait_event(ev)
                    if wire:
                        for i in range(a, b):
                            ctx.unpack48(din[i], dcts[i])
                    ctx.hrot_batch(evks[a:b], dcts[a:b], LEVEL, rs[a:b], outs[a:b])
                    if wire:
                        for i in range(a, b):
                            ctx.pack48(outs[i], dout[i])
                    done = torch.cuda.Event()
                    done.record(cur)
                    d2h_s.wait_event(done)
                    with torch.cuda.stream(d2h_s):
                        for i in range(a, b):
                            hout[i].copy_(dout[i], non_blocking=True)
                cur.wait_stream(d2h_s)

            return e2e_step, sum(h.numel() * 8 for h in hin)

        res = {}
        for wire in (True, False):
            fn, nb = make_step(wire)
            ms_e, _ = timed(fn, max(1, args.steps // 2), 1)
            res[wire] = (ms_e, nb)
        (ms_e2e, nb), (ms_u, nb_u) = res[True], res[False]
        e2e = {"value": BATCH * ws * 1000.0 / ms_e2e, "unit": UNIT, "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "ms_per_step": ms_e2e,
               "note": f"H2D of the 64 input ciphertexts from pinned memory in the 48-bit wire format (hy_pack48), "
                       f"unpack, hrot_batch, pack, D2H of the 64 outputs, in chunks of {E2E_CHUNK} with the copies "
                       "on two side streams (overlapped with the key switching); evaluation keys are server "
                       "state, resident before timing (P:1030)",
               "u64_words": {"value": BATCH * ws * 1000.0 / ms_u, "ms_per_step": ms_u, "h2d_bytes_per_step": nb_u,
                             "d2h_bytes_per_step": nb_u, "note": "the same with one uint64 per residue"}}

    conv = conv18 = blocks = None
    if not args.no_conv:
        del evks, cts, outs, houts
        torch.cuda.empty_cache()
        rates = (41000.0, 30000.0)
        if variants:
            rates = (variants["l+1=10"]["hoisted"]["keyswitch_per_s"], variants["l+1=7"]["plain"]["keyswitch_per_s"])
        conv = bench_conv(ctx, ws, rank, max(2, args.steps // 2), 1, timed, rates=rates)
        conv18 = None if args.no_r18 else bench_conv(ctx, ws, rank, 2, 1, timed, R18_LAYERS, "ResNet-18", rates)
        blocks = bench_blocks(ctx, ws, rank, max(2, args.steps // 2), 1, timed)

    boot = None
    if not args.no_conv:
        boot = bench_boot_linear(ctx, max(3, args.steps), 2, timed)


    c1 = None
    if not args.no_c1:
        c1 = bench_c1(local, max(3, args.steps), 2, timed, with_oracle=ws == 1 and not args.no_cpu_baseline)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        nproc = os.cpu_count()
        rate, dt = oracle_rate_threads(args.cpu_rotations, nproc)
        rate1, dt1 = oracle_rate_threads(max(1, args.cpu_rotations // 15), 1)
        cpu = {"value": rate, "unit": UNIT, "cores": nproc, "kind": "oracle", "cpu_model": cpu_model(),
               "sample": f"{args.cpu_rotations} plain HRot(s) at full level (Set_hyp, N=2^16), {dt:.1f} s, "
                         f"OMP_NUM_THREADS={nproc}",
               "one_thread": {"value": rate1, "unit": UNIT, "cores": 1,
                              "sample": f"{max(1, args.cpu_rotations // 15)} plain HRot(s), {dt1:.1f} s, "
                                        "OMP_NUM_THREADS=1"}}
        if c1 is not None:
            cpu["c1"] = {"oracle_ms": c1.get("oracle_ms"), "gpu_ms": c1["ms"], "cores": nproc}
        if conv is not None:  # the same ResNet-20 layers, whole, through the oracle beside the GPU times
            lay = oracle_conv_layers()
            for nm, x in lay.items():
                x["gpu_ms"] = conv["layers"][nm]["ms"]
                x["oracle_over_gpu"] = x["oracle_ms"] / x["gpu_ms"]
            cpu["resnet20_layers"] = {"layers": lay, "cores": os.cpu_count(),
                                      "sample": "whole layers (every output ct), oracle EncConv on the host cores"}
        if conv18 is not None:
            x = oracle_conv_layer_extrapolated("L2_ds")
            x["gpu_ms"] = conv18["layers"]["L2_ds"]["ms"]
            x["oracle_over_gpu"] = x["oracle_ms_extrapolated"] / x["gpu_ms"]
            cpu["resnet18_layer"] = x

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": "C2 HRot keyswitch microbenchmark, N=2^16, Set_hyp L+1=24 dnum=6 K=4, "
                                   "batch of 64 plain (non-hoisted) rotations per step per GPU",
                       "global_batch": BATCH * ws, "level": LEVEL, "parallelism": f"independent batches x{ws}",
                       "l2": "inputs larger than L2 (64 x 126 MiB packed evaluation keys streamed per step)"},
            "roofline": roof,
            "roofline_families": roofs,
            "roofline_hoisted": roofs_hoisted,
            "hrot_hbm": hrot_hbm,
            "resnet20_conv": conv,
            "resnet18_conv": conv18,
            "resnet20_blocks": blocks,
            "c1_raconv": c1,
            "boot_linear_f4": boot,
            "keyset_f2": keyset_report(),
            "plan_search_f3": plan_search_report(),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches * args.steps,  # our kernels launched inside the timed region (K steps)
            "gpu_launches_per_step": launches,
            "clocks": clocks,
            "hrot_variants": variants,
            "hoisted": {"value": BATCH * ws * 1000.0 / ms_h, "unit": UNIT, "ms_per_step": ms_h,
                        "note": "ct_0 rotated by 1..64 with one shared ModUp (Slide_f pattern, P:369-375)",
                        "kernel_breakdown": breakdown_h},
            "kernel_breakdown": breakdown,
            "ntt_ms_per_step": ntt_ms,
        }
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rotations", type=int, default=60)
    ap.add_argument("--no-conv", action="store_true", help="skip the ResNet-20 / ResNet-18 conv-layer timings")
    ap.add_argument("--no-r18", action="store_true", help="skip the ResNet-18 (PRCR) conv-layer timings")
    ap.add_argument("--no-variants", action="store_true", help="skip the HRot variant x level table")
    ap.add_argument("--no-c1", action="store_true", help="skip the BASELINE configs[0] RAConv timing")
    args = ap.parse_args()
    if args.impl == "reference":  # the CPU oracle on rank 0; no process group (the other ranks exit 0 at once)
        run_reference(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    ws, rank, local = dist_setup()
    run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
