"""(m, d) plan search for a HyPHEN network ("Parameter Study", tb:Rot and Boot).

HyPHEN's 2D-gap packing is parameterised per stage by (m, d) of CAConv's input format CA(m, d): the
choice fixes the rotation counts of every conv layer (table "Cost of homomorphic convolutions") and the
number of bootstrappings ("2D gap packing method helps balance the amount of rotation and
bootstrapping").  This module enumerates the stage formats the product implements, counts each plan's conv
rotations with the product's own layer plans (hy_conv_plan_create / hy_conv_plan_query, host only) and its
bootstrappings with the paper's block structure, and ranks the plans by a per-operation cost model.

Bootstrapping count (DESIGN R-BOOT): one bootstrapping per ciphertext entering a residual block, plus one --
    boots = 1 + sum over blocks of n_ct(block input),  n_ct = ceil(c / (c_n m)),  c_n = (N/2) / (e W_p^2),
    e = m d / g^2.
This reproduces all four Boot entries of tb:Rot and Boot that name an (m, d) plan: 10 (ResNet-20 Optimal),
15 (ResNet-20 Min Rot), 65 (ResNet-18 Optimal), 38 (ResNet-18 Min Boot) (tests/test_planner_cpu.py).

Implementable stage sequences: the product's stride-2 CAConv maps CA(m, d) at gap g to RA(2d, 2m) at gap 2g and
needs m = g (DESIGN R-DSCONV), so a network's plan is fixed by stage 1's d (m_1 = g_1 = 1): stage s runs at
(2^(s-1), 2^(s-1) d_1).  The paper's other rows (Min Rot, Min Boot) change (m, d) differently at a downsampling
layer (their IR figures are lost): their bootstrap counts are exact here, their conv rotations are not
modelled.

Cost model (context: the paper's CPU per-operation times, tb:Benchmark P:148): t = rotations x CRot + boots x Boot
+ PMults x MulPt.  The search keeps the implementable plan of least modelled time.
"""
from __future__ import annotations

from dataclasses import dataclass, field

# tb:Benchmark, ms per operation on the paper's 64-thread CPU
PAPER_CPU_MS = {"CRot": 15.5, "Boot": 2160.0, "MulPt": 0.506}


@dataclass
class Net:
    """A ResNet: per stage (channels, image width) and blocks; W_p the physical width; stage 1 has no DS block."""
    name: str
    stages: list            # [(channels, width, n_blocks)]
    wp: int
    stem: tuple | None = None   # (c_in, c_out) of a stem conv run in stage 1's format (ResNet-20), or None
    prcr: int = 1               # PRCR |S| of the stride-1 layers (ResNet-18: 8)


RESNET20 = Net("ResNet-20", [(16, 32, 3), (32, 16, 3), (64, 8, 3)], 32, stem=(3, 16))
RESNET18 = Net("ResNet-18", [(64, 56, 2), (128, 28, 2), (256, 14, 2), (512, 7, 2)], 64, prcr=8)


def n_ct(c: int, m: int, d: int, g: int, wp: int, n: int) -> int:
    """ciphertexts of a c-channel tensor in CA(m, d) at gap g (DESIGN R-LAYOUT)"""
    e = m * d // (g * g)
    cn = n // (e * wp * wp)
    per = cn * m
    return -(-c // per)


def boots(net: Net, fmts: list, n: int = 1 << 15) -> int:
    """DESIGN R-BOOT: 1 + sum over residual blocks of the ciphertexts entering the block (a DS block's input is in
    the previous stage's format)."""
    total = 1
    for s, ((c, w, nb), (m, d)) in enumerate(zip(net.stages, fmts)):
        g = 1 << s
        for b in range(nb):
            if s > 0 and b == 0:
                pc, _, _ = net.stages[s - 1]
                pm, pd = fmts[s - 1]
                total += n_ct(pc, pm, pd, g // 2, net.wp, n)
            else:
                total += n_ct(c, m, d, g, net.wp, n)
    return total


@dataclass
class PlanCost:
    fmts: list
    rotations: int = 0
    pmults: int = 0
    boots: int = 0
    layers: list = field(default_factory=list)   # (layer, multiplicity, rotations, pmults, counts by tag)
    feasible: bool = True
    why: str = ""

    def time_ms(self, ms=PAPER_CPU_MS):
        return self.rotations * ms["CRot"] + self.boots * ms["Boot"] + self.pmults * ms["MulPt"]


def _plan(ConvPlan, log_n, *spec, S=1):
    return ConvPlan(None, *spec, log_n=log_n, S=S)


def evaluate(net: Net, fmts: list, log_n: int = 16) -> PlanCost:
    """conv rotations / PMults of every layer of `net` in stage formats fmts (the product's layer plans, host only)
    and the bootstrapping count; infeasible when a layer has no plan in this product (HyError)."""
    from . import ConvPlan, HyError
    pc = PlanCost(fmts=list(fmts), boots=boots(net, fmts, 1 << (log_n - 1)))
    wp = net.wp
    try:
        for s, ((c, w, nb), (m, d)) in enumerate(zip(net.stages, fmts)):
            g = 1 << s
            # PRCR where its preconditions hold (DESIGN R-PRCR: e = 1, |S| | W_p/g, padding room)
            S = net.prcr if (m * d == g * g and (wp // g) % net.prcr == 0 and (wp // g) >= w + 1) else 1
            layers = []
            if s == 0 and net.stem:
                layers.append(("stem", 1, (net.stem[0], net.stem[1], w, 3, 1, wp, g, m, d, "CA"), 1))
            n_ca = nb if s == 0 else nb - 1
            n_ra = nb
            layers.append((f"L{s + 1}_ca", n_ca, (c, c, w, 3, 1, wp, g, m, d, "CA"), S))
            layers.append((f"L{s + 1}_ra", n_ra, (c, c, w, 3, 1, wp, g, d, m, "RA"), S))
            if s > 0:
                pcn, pw, _ = net.stages[s - 1]
                pm, pd = fmts[s - 1]
                if (m, d) != (2 * pm, 2 * pd) or pm != g // 2:
                    pc.feasible, pc.why = False, f"stage {s + 1}: (m, d) = {(m, d)} is not the R-DSCONV image of " \
                                                 f"{(pm, pd)} (needs m = g and (2m, 2d))"
                    return pc
                layers.append((f"L{s + 1}_ds", 1, (pcn, c, pw, 3, 2, wp, g // 2, pm, pd, "CA"), 1))
                layers.append((f"L{s + 1}_pconv", 1, (pcn, c, pw, 1, 2, wp, g // 2, pm, pd, "CA"), 1))
            for name, mult, spec, S_ in layers:
                p = _plan(ConvPlan, log_n, *spec, S=S_)
                rot = sum(p.counts[k] for k in ("Slide", "RaS", "RaS_g", "IR_g"))
                pc.rotations += mult * rot
                pc.pmults += mult * p.counts["PMult"]
                pc.layers.append((name, mult, rot, p.counts["PMult"], dict(p.counts)))
    except HyError as e:
        pc.feasible, pc.why = False, str(e)
    return pc


def candidates(net: Net, log_n: int = 16):
    """implementable stage sequences: m_1 = 1, d_1 a power of two, stage s at (2^(s-1), 2^(s-1) d_1)"""
    n = 1 << (log_n - 1)
    d1 = 1
    while d1 * net.wp * net.wp <= n:
        yield [(1 << s, (1 << s) * d1) for s in range(len(net.stages))]
        d1 *= 2


def search(net: Net, log_n: int = 16, ms=PAPER_CPU_MS):
    """every implementable plan with its counts and modelled time, best first"""
    out = [evaluate(net, f, log_n) for f in candidates(net, log_n)]
    out = [p for p in out if p.feasible]
    out.sort(key=lambda p: p.time_ms(ms))
    return out
