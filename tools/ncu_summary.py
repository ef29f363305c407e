"""Summarise ncu captures for profiles/ (read here, on the CPU box).

  python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --name r1_c2 [--config C2]
      -> profiles/ncu_<name>.md (per-kernel table) and updates profiles/ncu_traffic.json
  python tools/ncu_summary.py --launches gpurun_out/launches.csv --name r1_c2
      -> profiles/launches_<name>.md (per-kernel share of the launch list)

Kernel classes follow libhks's profiler names (hks_prof_read) so bench.py can attach the
`dram__bytes_read.sum + dram__bytes_write.sum` of its dominant kernel as roofline.traffic.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def kernel_class(name: str) -> str:
    if name.startswith("k_ntt_kip"):
        return "ntt_rows_kip"
    if name.startswith("k_bconv"):
        return "bconv"
    if name.startswith("k_kip"):
        return "kip"
    if name.startswith("k_automorph"):
        return "automorph"
    if name.startswith("k_intt_cl"):
        return "ntt_inv_fused"
    if name.startswith("k_evk_prepare"):
        return "setup: evk_prepare"
    if name.startswith("k_ntt<") or name.startswith("void k_ntt<"):
        args = name[name.index("<") + 1:name.index(">")].split(",")
        cols, fwd, epi = int(args[4]), int(args[5]), int(args[6])
        if fwd:
            return "ntt_fwd_cols" if cols else ("ntt_fwd_rows_moddown" if epi == 2 else "ntt_fwd_rows")
        return "ntt_inv_cols_scale" if cols else "ntt_inv_rows"
    return name


def metric(row, hdr, key):
    try:
        return float(row[hdr.index(key)])
    except (ValueError, IndexError):
        return float("nan")


def summarise_rep(rep, name, config):
    raw = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], text=True, stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    stall_keys = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")]
    out = []
    traffic = collections.defaultdict(list)
    for row in rows[2:]:
        kname = row[hdr.index("Kernel Name")].replace("void ", "")
        cls = kernel_class(kname)
        dram_r = metric(row, hdr, "dram__bytes_read.sum")
        dram_w = metric(row, hdr, "dram__bytes_write.sum")
        u = units[hdr.index("dram__bytes_read.sum")]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        tu = units[hdr.index("gpu__time_duration.sum")]
        tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(tu, 1.0)
        t_us = metric(row, hdr, "gpu__time_duration.sum") * tscale
        stalls = sorted(((metric(row, hdr, h), h.replace("smsp__average_warps_issue_stalled_", "")
                          .replace("_per_issue_active.ratio", "")) for h in stall_keys), reverse=True)[:3]
        rec = {
            "kernel": kname[:60], "class": cls, "time_us": t_us,
            "dram_read_MB": dram_r * scale / 1e6, "dram_write_MB": dram_w * scale / 1e6,
            "dram_GBps": (dram_r + dram_w) * scale / (t_us * 1e-6) / 1e9 if t_us else float("nan"),
            "issue_pct": metric(row, hdr, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "occupancy_pct": metric(row, hdr, "sm__warps_active.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": metric(row, hdr, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "alu_pipe_pct": metric(row, hdr, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
            "warp_inst_M": metric(row, hdr, "smsp__inst_executed.sum") / 1e6,
            "regs": metric(row, hdr, "launch__registers_per_thread"),
            "grid": metric(row, hdr, "launch__grid_size"),
            "top_stalls": ", ".join(f"{n}={v:.2f}" for v, n in stalls),
        }
        out.append(rec)
        traffic[cls].append((dram_r + dram_w) * scale)
    md = [f"# ncu --set full summary: {name}", "",
          f"Source: `{os.path.basename(rep)}` (cold-cache, serialised replays; compare shares and counters, "
          f"not absolute times).", "",
          "| kernel | class | time µs | DRAM R MB | DRAM W MB | DRAM GB/s | issue % | occ % | FMA % | ALU % | "
          "warp inst M | regs | grid | top stalls |", "|" + "---|" * 14]
    for r in out:
        md.append(f"| `{r['kernel']}` | {r['class']} | {r['time_us']:.1f} | {r['dram_read_MB']:.1f} | "
                  f"{r['dram_write_MB']:.1f} | {r['dram_GBps']:.0f} | {r['issue_pct']:.1f} | {r['occupancy_pct']:.1f} | "
                  f"{r['fma_pipe_pct']:.1f} | {r['alu_pipe_pct']:.1f} | {r['warp_inst_M']:.2f} | {r['regs']:.0f} | "
                  f"{r['grid']:.0f} | {r['top_stalls']} |")
    os.makedirs(PROF, exist_ok=True)
    with open(os.path.join(PROF, f"ncu_{name}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    tpath = os.path.join(PROF, "ncu_traffic.json")
    data = json.load(open(tpath)) if os.path.exists(tpath) else {}
    data.setdefault(config, {})
    for cls, v in traffic.items():
        data[config][cls] = sum(v) / len(v)          # mean DRAM bytes per launch of that class
    data.setdefault("_source", {})[config] = f"profiles/ncu_{name}.md"
    with open(tpath, "w") as f:
        json.dump(data, f, indent=1, sort_keys=True)
    print("\n".join(md))


def summarise_launches(path, name):
    rows = list(csv.reader(open(path)))
    # ncu --csv launch list: find the header line containing "Kernel Name"
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[start]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        unit = r[hdr.index("Metric Unit")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
        cls = kernel_class(r[hdr.index("Kernel Name")].replace("void ", ""))
        agg[cls][0] += 1
        agg[cls][1] += v
    # shares of the KeySwitch step: one-time setup kernels (key preparation at load time) are listed apart
    tot = sum(v[1] for c, v in agg.items() if not c.startswith("setup"))
    md = [f"# ncu launch list: {name}", "",
          "`ncu --metrics gpu__time_duration.sum --clock-control none` over bench.py (cold-cache, serialised).", "",
          "| kernel class | launches | total µs | share |", "|---|---|---|---|"]
    for cls, (n, t) in sorted(agg.items(), key=lambda kv: (kv[0].startswith("setup"), -kv[1][1])):
        md.append(f"| {cls} | {n} | {t:.1f} | " + ("outside the timed step" if cls.startswith("setup") else f"{t / tot:.3f}") + " |")
    with open(os.path.join(PROF, f"launches_{name}.md"), "w") as f:
        f.write("\n".join(md) + "\n")
    print("\n".join(md))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--name", required=True)
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    if a.rep:
        summarise_rep(a.rep, a.name, a.config)
    if a.launches:
        summarise_launches(a.launches, a.name)
