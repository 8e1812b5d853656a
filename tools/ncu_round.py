"""Build the committed profile evidence of a round from gpurun_out/ (written by tools/profile_round.sh):

    python tools/ncu_round.py <tag>

-> profiles/<tag>_ncu_summary.md  (launch-list shares + key metrics / stalls of each `--set full` capture)
-> profiles/<tag>_launches.csv    (copy of the raw launch list)
-> profiles/ncu_traffic.json      (dram read+write bytes per launch per kernel family; bench.py reports it
                                   as roofline.traffic)
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

# kernel-name prefix -> bench.py family (hy_internal.h Family)
FAMILY = [("k_rows_ip_final_tma<6, 1", "ntt_ip_hoisted"), ("k_rows_ip_final", "ntt_ip"),
          ("k_bconv_cols<4, 1", "moddown"), ("k_bconv_cols", "modup"), ("k_modup_cols", "modup"), ("k_modup_bconv", "modup"), ("k_ntt_rows_ip", "ntt_ip"),
          ("k_ntt_rows_final", "moddown"), ("k_moddown_bconv", "moddown"), ("k_moddown_final", "moddown"),
          ("k_ks_ip", "ip"), ("k_ntt_cols", "ntt_a"), ("k_ntt_rows", "ntt_b"), ("k_automorph", "aut")]
KEYS = ["Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def family(name):
    short = name.split("(")[0].split("::")[-1]
    if short.startswith("k_ntt_rows_ip") and short.endswith(", 1>"):  # <B, SUM, HOIST=1>: hoisted P-limb IP
        return "ntt_ip_hoisted", short
    if short.startswith("k_rows_ip_p_tma"):  # <B, HOIST>: the P-limb IP on the bulk-copy ring
        return ("ntt_ip_hoisted" if short.endswith(", 1>") or short.endswith(", true>") else "ntt_ip"), short
    # the hoisted step's one shared ModUp (separate NTT passes + BConv): not part of the plain step's families
    for pre, fam in (("k_modup_bconv", "modup_hoisted"), ("k_ntt_rows<", "ntt_b_hoisted"),
                     ("k_ntt_cols256", "ntt_a_hoisted")):
        if short.startswith(pre):
            return fam, short
    for pre, fam in FAMILY:
        if short.startswith(pre):
            return fam, short
    return None, short


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return dict(zip(r[0], r[2])), dict(zip(r[0], r[1]))


def launch_table(path):
    rows = list(csv.reader(l for l in open(path) if not l.startswith("==")))
    h = rows[0]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for x in rows[1:]:
        if len(x) != len(h) or x[mi] != "gpu__time_duration.sum":
            continue
        name = x[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("hy::", "")
        t = float(x[vi].replace(",", ""))
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += t
    return agg


def main():
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    md = [f"# {tag}: ncu evidence (B200, sm_100a)", "",
          "Produced by `tools/profile_round.sh " + tag + "` under gpurun and `tools/ncu_round.py " + tag + "`.",
          "Launch list: `ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none` over",
          "bench.py's timed regions (`HY_NCU_TIMED=1`, 1 plain step of 64 HRots + 1 hoisted step); the per-launch",
          "times are cold-cache and serialised, so compare shares, not absolutes.  Full captures: one launch per",
          "kernel, `--set full --clock-control none --import-source on` (64 key switches per launch, L+1 = 24).", ""]
    lpath = os.path.join(OUT, f"launches_{tag}.csv")
    if os.path.exists(lpath):
        shutil.copy(lpath, os.path.join(PROF, f"{tag}_launches.csv"))
        agg = launch_table(lpath)
        tot = sum(v[1] for v in agg.values())
        md += ["## Launch list", "```", f"total {tot / 1000:.1f} us, {sum(v[0] for v in agg.values())} launches",
               f"{'kernel':48s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            md.append(f"{k[:48]:48s} {n:8d} {t / 1000:10.1f} {100 * t / tot:5.1f}% {t / n / 1000:8.1f}")
        md += ["```", ""]
    traffic = {"source": f"profiles/{tag}_ncu_summary.md (ncu --set full, one launch per kernel)", "families": {}}
    fam_acc = collections.defaultdict(list)
    md += ["## Full captures"]
    for f in sorted(os.listdir(OUT)):
        if not (f.startswith(f"prof_{tag}_") and f.endswith(".ncu-rep")):
            continue
        d, units = raw(os.path.join(OUT, f))
        name = d.get("Kernel Name", f)
        fam, short = family(name)
        md += [f"### {short}", "```", f"{'Kernel Name':60s} {name[:100]}"]
        for k in KEYS:
            if k in d:
                md.append(f"{k:60s} {d[k]} {units.get(k, '')}")
        st = [(k, float(x.replace(",", ""))) for k, x in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued") and x]
        st = [(k, x) for k, x in st if x > 0]
        tot = sum(x for _, x in st) or 1.0
        md.append("stalls: " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * x / tot:.0f}%"
                                         for k, x in sorted(st, key=lambda t: -t[1])[:8]))
        md += ["```", ""]
        rd = float(d.get("dram__bytes_read.sum", "0").replace(",", ""))
        wr = float(d.get("dram__bytes_write.sum", "0").replace(",", ""))
        if fam:
            fam_acc[fam].append((short, rd + wr))
    for fam, lst in fam_acc.items():
        traffic["families"][fam] = {"kernel": " + ".join(k for k, _ in lst),
                                    "dram_bytes": sum(b for _, b in lst) / len(lst), "items": int(os.environ.get("HY_ITEMS", "64"))}
    with open(os.path.join(PROF, f"{tag}_ncu_summary.md"), "w") as fh:
        fh.write("\n".join(md) + "\n")
    with open(os.path.join(PROF, "ncu_traffic.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
