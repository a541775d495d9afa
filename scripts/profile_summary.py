"""Summarise a round's profiling artefacts into profiles/ (run here, no GPU).

usage: python scripts/profile_summary.py <launches.csv> <full.ncu-rep> <tag> <steps-in-launch-list> [config]
Writes profiles/<tag>_launches.md (per-kernel share of device time from the
ncu launch list) and profiles/<tag>_kernels.md + profiles/traffic_c4.json
(DRAM bytes per launch from the --set full capture, used by bench.py as
roofline.traffic)."""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
    return agg


def full(path):
    if path.endswith(".csv"):  # raw page exported on the GPU box (ncu -i rep --page raw --csv)
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    res = []
    for r in rows[2:]:
        d = dict(zip(h, r))
        def g(k):
            # section-prefixed names (e.g. "LTS.TriageCompute.lts__throughput...") are accepted too
            key = k if k in d else next((h_ for h_ in d if h_.endswith("." + k)), None)
            return float(d[key].replace(",", "")) if key and d[key] not in ("", "n/a") else None
        res.append({
            "kernel": d["Kernel Name"].split("(")[0].replace("void ", "").strip(),
            "grid": d.get("Grid Size"), "block": d.get("Block Size"),
            "time_ms": g("gpu__time_duration.sum"),
            "dram_read_GB": (g("dram__bytes_read.sum") or 0) / 1e9 * (1e3 if d.get("dram__bytes_read.sum", "").count(".") == 0 else 1),
            "dram_bytes_read": g("dram__bytes_read.sum"), "dram_bytes_write": g("dram__bytes_write.sum"),
            "dram_pct": g("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
            "fp64_pct": g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
            "l1_pct": g("l1tex__throughput.avg.pct_of_peak_sustained_active"),
            "lsu_pct": g("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
            "issue_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "regs": g("launch__registers_per_thread"),
            "smem_wf": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
            "smem_conf": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
            "cycles": g("sm__cycles_active.avg"),
            "l2_bytes": g("l1tex__m_xbar2l1tex_read_bytes.sum"),
            "l2_pct": g("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "l2_hit": g("lts__t_sector_op_read_hit_rate.pct"),
            "l2x_bps": g("derived__lts__lts2xbar_bytes.sum.per_second"),
            "stalls": sorted(((g(k) or 0.0, k.replace("smsp__average_warps_issue_stalled_", "").replace(
                "_per_issue_active.ratio", "")) for k in d if k.startswith("smsp__average_warps_issue_stalled_")
                and k.endswith("_per_issue_active.ratio") and "selected" not in k), reverse=True)[:3],
        })
    units = dict(zip(rows[0], rows[1]))
    return res, units


def main(lpath, fpath, tag, steps, config="c4"):
    os.makedirs(os.path.join(REPO, "profiles"), exist_ok=True)
    agg = launches(lpath)
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(REPO, "profiles", f"{tag}_{config}_launches.md"), "w") as f:
        f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none; cold-cache, serialised)\n\n")
        f.write(f"Command: `ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none "
                f"python scripts/profile_step.py {config}` (scripts/gpu_profile.sh): exactly {steps} bench step(s) "
                "(refined type-5 + refined type-4) after 3 warm-up steps; compare SHARES with bench.py's live "
                "kernels_ms_per_step.\n\n")
        f.write("| kernel | launches | total ms | share |\n|---|---|---|---|\n")
        for k, (n, ns) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| `{k}` | {n} | {ns / 1e6:.3f} | {ns / tot * 100:.1f}% |\n")
    res, units = full(fpath)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    ur, uw = scale.get(units.get("dram__bytes_read.sum", "byte"), 1), scale.get(units.get("dram__bytes_write.sum", "byte"), 1)
    ul = scale.get(units.get("l1tex__m_xbar2l1tex_read_bytes.sum", "byte"), 1)
    traffic = collections.defaultdict(list)
    tunit = units.get("gpu__time_duration.sum", "msecond")
    tscale = {"msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "ms": 1.0, "us": 1e-3, "ns": 1e-6}.get(tunit, 1.0)
    with open(os.path.join(REPO, "profiles", f"{tag}_{config}_kernels.md"), "w") as f:
        f.write(f"# {tag}: ncu --set full captures ({config}, one bench step)\n\n")
        f.write("LSU pipe % = `l1tex__data_pipe_lsu_wavefronts` (shared + global + local wavefronts of the one L1 data "
                "pipe, % of its peak: the resource that bounds the two-FFT chain kernels and the gridding kernels); "
                "Shared-memory busy = LSU shared wavefronts / (SMs x active cycles); L2->SM GB = "
                "`l1tex__m_xbar2l1tex_read_bytes.sum` (bytes the SMs read from L2; writes go through to L2 as "
                "well), its rate over the kernel time, `lts__throughput` % of peak (the busiest L2 sub-unit) and "
                "the L2 read-sector hit rate; stalls = top three `smsp__average_warps_issue_stalled_*` per issued "
                "instruction.\n\n")
        f.write("| kernel | grid | ms | DRAM read GB | DRAM write GB | DRAM % peak | L2->SM GB | L2->SM GB/s | L2 % peak | L2 read hit % "
                "| fp64 pipe % | L1 % | LSU pipe % | SMEM busy % | bank conflicts % | issue % | warps active % | regs | top stalls |\n")
        f.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in res:
            rb, wb = (r["dram_bytes_read"] or 0) * ur, (r["dram_bytes_write"] or 0) * uw
            traffic[r["kernel"]].append(rb + wb)
            smem = 100.0 * (r["smem_wf"] or 0) / 148 / r["cycles"] if r["cycles"] else 0.0
            conf = 100.0 * (r["smem_conf"] or 0) / r["smem_wf"] if r["smem_wf"] else 0.0
            st = ", ".join(f"{n} {v:.2f}" for v, n in r["stalls"])
            lb = (r["l2_bytes"] or 0) * ul
            ms = r["time_ms"] * tscale
            l2 = (f"{lb / 1e9:.3f} | {lb / (ms / 1e3) / 1e9:.0f} | {r['l2_pct'] or 0:.1f} | {r['l2_hit'] or 0:.1f}"
                  if r["l2_bytes"] is not None else "— | — | — | —")
            f.write(f"| `{r['kernel']}` | {r['grid']} | {ms:.3f} | {rb / 1e9:.3f} | {wb / 1e9:.3f} | "
                    f"{r['dram_pct']:.1f} | {l2} | {r['fp64_pct']:.1f} | {r['l1_pct']:.1f} | {r['lsu_pct'] or 0:.1f} | {smem:.1f} | {conf:.1f} | "
                    f"{r['issue_pct']:.1f} | {r['warps_active_pct']:.1f} | {r['regs']:.0f} | {st} |\n")
    short = {}
    for k, v in traffic.items():
        key = {"kbm_pad": "bm_pad", "kbm_band": "bm_band", "kbm_mid": "bm_mid", "kbm_col": "bm_col", "kbm_row": "bm_row",
               "k_spread_p": "spread_p", "k_gather_b": "gather_b", "k_gather_p": "gather_p", "kbm_colin": "bm_colin",
               "kbm_rowout": "bm_rowout", "kc_col": "chain_col", "kc_band": "chain_band", "kc_mid": "chain_mid",
               "kc_pad": "chain_pad", "kc_row": "chain_row", "k_spread_s": "spread_s1",
               "k_gather_s": "gather_s1"}
        base = k.split("<")[0]
        for suf in ("_hst", "_hs", "_hf", "_hp", "_h", "_s"):  # hybrid / fused / persistent / TMA-store variants report under the stage's name
            if base.startswith("kbm_") and base.endswith(suf):
                base = base[: -len(suf)]
                break
        key = key.get(base, base)
        short.setdefault(key, []).extend(v)
    short = {k: sum(v) / len(v) for k, v in short.items()}  # mean over all launches of the stage
    json.dump(short, open(os.path.join(REPO, "profiles", f"traffic_{config}.json"), "w"), indent=1)
    print(json.dumps(short, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), *(sys.argv[5:6]))
