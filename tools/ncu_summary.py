"""Summarise an `ncu --set full` report: per kernel (first launch of each name)
duration, DRAM bytes, instructions, issue/occupancy and the top stall reasons.

    python tools/ncu_summary.py report.ncu-rep summary.txt traffic.json
"""
import csv, io, json, subprocess, sys

rep, out_txt, out_json = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
idx = {h: i for i, h in enumerate(hdr)}
stall = [h for h in hdr if h.startswith("smsp__average_warps_issue_stalled_")
         and h.endswith("_per_issue_active.ratio")]


def num(d, k):
    try:
        return float(d[idx[k]])
    except (KeyError, ValueError):
        return float("nan")


# pipe utilisation and shared-memory throughput (north_star: SM/LSU and shared-memory
# throughput for rasterization)
PIPES = (("fma_cycles", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
         ("fma_inst", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active"),
         ("alu", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active"),
         ("lsu", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"),
         ("xu", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
         ("fp64", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"))
SMEM = "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"
CONFL = "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"

lines, traffic, seen = [], {}, set()
for d in rows[2:]:
    name = d[idx["Kernel Name"]].split("(")[0].replace("uws::<unnamed>::", "").replace("void ", "")
    name = name.replace("radix::", "").replace("uws::", "").replace("(anonymous namespace)::", "")
    if name in seen:
        continue
    seen.add(name)
    t_us = num(d, "gpu__time_duration.sum")
    dram = (num(d, "dram__bytes_read.sum") + num(d, "dram__bytes_write.sum")) * 1e6  # MB -> B
    traffic[name] = {"time_us": t_us, "dram_bytes": dram}
    st = sorted(((num(d, h), h) for h in stall), reverse=True)[:4]
    lines.append(
        f"{name:32s} {t_us:9.1f} us  dram {dram / 1e6:8.1f} MB ({dram / max(t_us, 1e-9) / 1e3:7.1f} GB/s)"
        f"  inst {num(d, 'smsp__inst_executed.sum') / 1e6:7.1f} M  issue "
        f"{num(d, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}%  warps "
        f"{num(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  regs "
        f"{d[idx['launch__registers_per_thread']]:>3}\n      stalls: " +
        ", ".join(f"{h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}"
                  f"={v:.2f}" for v, h in st) +
        "\n      pipes (% of peak, active): " + ", ".join(
            f"{lbl}={num(d, m):.1f}" for lbl, m in PIPES) +
        f"; smem wavefronts {num(d, SMEM):.1f}% (bank conflicts {num(d, CONFL):.0f})")
with open(out_txt, "w") as f:
    f.write(f"ncu --set full --clock-control none (single launches, cold cache, serialised); {rep}\n")
    f.write("\n".join(lines) + "\n")
with open(out_json, "w") as f:
    json.dump(traffic, f, indent=1)
print("\n".join(lines))
