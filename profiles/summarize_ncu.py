#!/usr/bin/env python3
"""Summarise ncu reports into profiles/ncu_summary.json (+ .md), read by bench.py's roofline.

    python profiles/summarize_ncu.py gpurun_out/step_full.ncu-rep [more.ncu-rep ...]

Per kernel launch: duration, DRAM bytes read/written (the roofline "traffic"), issue-slot
utilisation, IPC, occupancy, registers, L2 hit rate and the top warp-stall reasons.  Kernel
names are mapped to the launch names bench.py's per-kernel profile uses.
"""
import csv
import io
import json
import re
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent

NAME_MAP = [  # (regex on the demangled ncu kernel name, bench launch name)
    (r"blend_backward", "blend_backward"),
    (r"blend_forward", "blend_forward"),
    (r"chain_touched_kernel", "chain"),
    (r"chain_compact_kernel", "chain_compact"),
    (r"chain_kernel", "chain"),
    (r"preprocess_kernel", "preprocess"),
    (r"adam_kernel", "adam"),
    (r"st_chunk_kernel<(\(bool\))?0", "st_count"),
    (r"st_chunk_kernel<(\(bool\))?1", "st_emit"),
    (r"bin_count_kernel", "bin_count"),
    (r"bin_emit_kernel", "bin_emit"),
    (r"bin_map_kernel", "bin_map"),
    (r"radix_coop_kernel", "radix_sort"),
    (r"radix_onesweep_kernel", "radix_onesweep"),
    (r"radix_histogram_kernel", "radix_histogram"),
    (r"scan_lookback_kernel", "scan"),
    (r"seg_setup_kernel", "seg_setup"),
    (r"loss_reduce_kernel", "loss_reduce"),
    (r"publish_counts_kernel", "publish_counts"),
    (r"st_ranges_from_chunks_kernel", "st_ranges"),
    (r"ranges_from_slots_kernel", "tile_ranges"),
    (r"quat_normalize_kernel", "quat_normalize"),
]

RAW = {
    "duration_ns": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "issue_active": "sm__instruction_throughput.avg.pct_of_peak_sustained_active",
    "occupancy": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "l2_hit": "lts__t_sector_hit_rate.pct",
    "inst": "smsp__inst_executed.sum",
    # pipe utilisation (% of peak, active cycles) and SIMT efficiency (threads per warp instruction)
    "pipe_fma": "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "pipe_alu": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "pipe_xu": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "pipe_lsu": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "fma_cycles": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "simt": "smsp__thread_inst_executed_per_inst_executed.ratio",
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
              "nsecond": 1, "usecond": 1e3, "msecond": 1e6}


def bench_name(kernel):
    for pat, name in NAME_MAP:
        if re.search(pat, kernel):
            return name
    return kernel.split("(")[0].split("<")[0].split("::")[-1]


def raw_rows(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    return [(dict(zip(head, r)), dict(zip(head, units))) for r in rows[2:] if len(r) == len(head)]


def num(row, units, key):
    v = row.get(key, "").replace(",", "")
    try:
        x = float(v)
    except ValueError:
        return None
    return x * UNIT_SCALE.get(units.get(key, ""), 1)


def summarise(reps):
    kernels = {}
    for rep in reps:
        for row, units in raw_rows(rep):
            name = bench_name(row.get("Kernel Name", "?"))
            d = {k: num(row, units, m) for k, m in RAW.items()}
            stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): num(row, units, k) or 0.0
                      for k in row if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
            tot = sum(stalls.values()) or 1.0
            top = sorted(stalls.items(), key=lambda kv: -kv[1])[:5]
            e = kernels.setdefault(name, {"launches": 0, "duration_us": 0.0, "dram_bytes": 0.0, "source": Path(rep).name,
                                          "kernel": row.get("Kernel Name", "")[:160]})
            e["launches"] += 1
            e["duration_us"] += (d["duration_ns"] or 0) / 1e3
            e["dram_bytes"] += (d["dram_read"] or 0) + (d["dram_write"] or 0)
            for k in ("ipc", "issue_active", "occupancy", "registers", "l2_hit", "inst", "pipe_fma", "pipe_alu", "pipe_xu",
                      "pipe_lsu", "fma_cycles", "simt"):
                if d[k] is not None:
                    e[k] = d[k]
            e["top_stalls"] = {k: round(v / tot, 3) for k, v in top}
    for e in kernels.values():
        e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
        e["duration_us_per_launch"] = e["duration_us"] / e["launches"]
        e["dram_gbs"] = e["dram_bytes"] / (e["duration_us"] * 1e3) if e["duration_us"] else None
    return kernels


def main(reps):
    kernels = summarise(reps)
    path = HERE / "ncu_summary.json"
    old = {"kernels": kernels, "sources": [Path(r).name for r in reps]}
    old["note"] = ("ncu --set full --clock-control none captures (cold caches, serialised replays): use shares and "
                   "per-launch DRAM bytes, not absolute times; regenerate with profiles/summarize_ncu.py")
    path.write_text(json.dumps(old, indent=1, sort_keys=True) + "\n")
    lines = ["| kernel | launches | us/launch | DRAM MB/launch | DRAM GB/s | issue % | IPC | occ % | regs | FMA pipe % | "
             "ALU % | XU % | LSU % | SIMT (thr/inst) | top stalls |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for name, e in sorted(old["kernels"].items(), key=lambda kv: -kv[1]["duration_us"]):
        st = ", ".join(f"{k} {v:.0%}" for k, v in e.get("top_stalls", {}).items())
        lines.append(f"| {name} | {e['launches']} | {e['duration_us_per_launch']:.1f} | "
                     f"{e['dram_bytes_per_launch'] / 1e6:.1f} | {e['dram_gbs'] or 0:.0f} | "
                     f"{e.get('issue_active', 0):.1f} | {e.get('ipc', 0):.2f} | {e.get('occupancy', 0):.1f} | "
                     f"{e.get('registers', 0):.0f} | {e.get('pipe_fma') or 0:.1f} | {e.get('pipe_alu') or 0:.1f} | "
                     f"{e.get('pipe_xu') or 0:.1f} | {e.get('pipe_lsu') or 0:.1f} | {e.get('simt') or 0:.1f} | {st} |")
    (HERE / "ncu_summary.md").write_text("# ncu --set full summary (per launch)\n\n" + "\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1:])
