"""Summarise an ncu --set full report (and optionally a launch list) into
profiles/: a markdown table and profiles/ncu_summary.json (read by bench.py
for the roofline `traffic` field).

    python scripts/ncu_summarize.py gpurun_out/full_C2_r1.ncu-rep C2 r1 [gpurun_out/launches_C2_r1.csv]
"""
import collections
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
PROF = ROOT / "profiles"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct"),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
    ("l1tex__t_sector_hit_rate.pct", "l1_hit_pct"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2_throughput_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_throughput_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem_wavefront_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "smem_ld_wavefronts"),
    ("smsp__sass_inst_executed_op_shared_ld.sum", "smem_ld_instr"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64_pipe_pct"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_pct"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu_pipe_pct"),
    ("launch__registers_per_thread", "registers"),
    ("smsp__inst_executed.sum", "warp_instructions"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}


def short(name):
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
    return name.split("(")[0]


def read_report(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    kernels = []
    for row in data:
        k = {"kernel": short(row[hdr.index("Kernel Name")])}
        for m, key in METRICS:
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            k[key] = v * SCALE.get(units[i], 1.0) if units[i] in SCALE else v
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(row[i])
                except ValueError:
                    pass
        k["top_stalls"] = sorted(((v, s) for s, v in stalls.items() if s != "selected"), reverse=True)[:3]
        if "dram_read" in k and "dram_write" in k:
            k["dram_bytes"] = k["dram_read"] + k["dram_write"]
            k["dram_GBps"] = k["dram_bytes"] / k["duration"] / 1e9
        if k.get("smem_ld_instr"):
            k["smem_wavefronts_per_ld"] = k["smem_ld_wavefronts"] / k["smem_ld_instr"]
        kernels.append(k)
    return kernels


def read_launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if r[mi] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
            tot[short(r[ki])] += v
            cnt[short(r[ki])] += 1
    T = sum(tot.values())
    return [(k, cnt[k], v, v / T) for k, v in sorted(tot.items(), key=lambda x: -x[1])]


def main():
    rep, cfg, tag = Path(sys.argv[1]), sys.argv[2], sys.argv[3]
    launches = sys.argv[4] if len(sys.argv) > 4 else None
    kernels = read_report(rep)
    lines = [f"# ncu summary -- {cfg} ({tag})", "",
             f"Source: `ncu --set full --clock-control none` of `scripts/profile_sigma.py {cfg} 1` "
             f"(report `{rep.name}`, not committed; 1 launch each, replayed ~40x, cold L2 per replay).", "",
             "| kernel | ms | DRAM bytes | DRAM GB/s | L2 hit % | L1 hit % | L2 thru % | L1tex thru % | smem wf % | "
             "wf/LDS | issue % | occ % | FP64 pipe % | tensor % | regs | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    summary = json.loads((PROF / "ncu_summary.json").read_text()) if (PROF / "ncu_summary.json").exists() else {}
    cfg_sum = summary[cfg] = {}   # this capture replaces the config's entry
    for k in kernels:
        f = lambda key, fmt="{:.1f}": fmt.format(k[key]) if key in k else "-"  # noqa: E731
        stalls = ", ".join(f"{s} {v:.1f}" for v, s in k["top_stalls"])
        lines.append(f"| {k['kernel']} | {k['duration'] * 1e3:.2f} | {f('dram_bytes', '{:.3g}')} | {f('dram_GBps')} | "
                     f"{f('l2_hit_pct')} | {f('l1_hit_pct')} | {f('l2_throughput_pct')} | {f('l1tex_throughput_pct')} | "
                     f"{f('smem_wavefront_pct')} | {f('smem_wavefronts_per_ld', '{:.2f}')} | {f('issue_active_pct')} | "
                     f"{f('occupancy_pct')} | {f('fp64_pipe_pct')} | {f('tensor_pipe_pct')} | {f('registers', '{:.0f}')} | {stalls} |")
        name = k["kernel"]
        if name not in cfg_sum or k["duration"] > cfg_sum[name].get("duration", 0):
            cfg_sum[name] = {kk: vv for kk, vv in k.items() if kk != "top_stalls"}
            cfg_sum[name]["report"] = f"{rep.name} ({tag})"
    if launches:
        lines += ["", f"## Launch list (`ncu --metrics gpu__time_duration.sum` of `bench.py --config {cfg} --steps 2`)",
                  "", "Serialised and cold-cache per launch: compare shares, not absolutes.", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, n, v, s in read_launches(launches):
            lines.append(f"| {k} | {n} | {v * 1e3:.2f} | {s:.3f} |")
    (PROF / f"ncu_{cfg}_{tag}.md").write_text("\n".join(lines) + "\n")
    (PROF / "ncu_summary.json").write_text(json.dumps(summary, indent=1))
    print("\n".join(lines))


if __name__ == "__main__":
    main()
