"""(m, d) plan search, host only: the bootstrapping model reproduces the paper's
Boot column for every plan of tb:Rot and Boot that names its (m, d), and the search over the product's
implementable plans, under the paper's own per-operation CPU costs (tb:Benchmark P:148), selects the plans the
paper reports as Optimal for both networks."""
import pytest

from paper_2302_02407_b200 import planner as P


@pytest.mark.parametrize("net,fmts,want", [
    (P.RESNET20, [(1, 2), (2, 4), (4, 8)], 10),              # ResNet-20 Optimal
    (P.RESNET20, [(1, 2), (1, 8), (2, 16)], 15),             # ResNet-20 Min Rot
    (P.RESNET18, [(1, 1), (2, 2), (4, 4), (8, 8)], 65),      # ResNet-18 Optimal
    (P.RESNET18, [(1, 1), (4, 1), (16, 1), (64, 1)], 38),    # ResNet-18 Min Boot
])
def test_boot_model_matches_paper(net, fmts, want):
    assert P.boots(net, fmts) == want


def test_search_selects_paper_optimal():
    best20 = P.search(P.RESNET20)[0]
    assert best20.fmts == [(1, 2), (2, 4), (4, 8)] and best20.boots == 10
    # SISO (Slide) rotations of the plan = the paper's 152 (19 3x3 convs incl. the stem x 8)
    assert sum(mult * c["Slide"] for name, mult, _, _, c in best20.layers if not name.endswith("pconv")) == 152
    best18 = P.search(P.RESNET18)[0]
    assert best18.fmts == [(1, 1), (2, 2), (4, 4), (8, 8)] and best18.boots == 65
    # the modelled CPU time of the chosen ResNet-20 plan is within 5 % of the paper's measured 37.57 s
    assert abs(best20.time_ms() / 1000 - 37.57) / 37.57 < 0.05


def test_search_trades_rotations_for_boots():
    """a plan with fewer rotations can lose on bootstrapping -- ResNet-20 d_1 = 4 needs fewer conv
    rotations than the Optimal plan but almost twice the bootstrappings, and ranks below it"""
    plans = {tuple(p.fmts[0]): p for p in P.search(P.RESNET20)}
    assert plans[(1, 4)].rotations < plans[(1, 2)].rotations
    assert plans[(1, 4)].boots > plans[(1, 2)].boots
    assert plans[(1, 4)].time_ms() > plans[(1, 2)].time_ms()


def test_infeasible_transition_reported():
    pc = P.evaluate(P.RESNET20, [(1, 2), (1, 8), (2, 16)])
    assert not pc.feasible and "R-DSCONV" in pc.why
