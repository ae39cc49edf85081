"""Summarise one `ncu --set full` report (first kernel) into a JSON dict for profiles/."""
import csv, json, subprocess, sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6, "ns"),
    "dram_bytes_read": ("dram__bytes_read.sum", 1, "byte"),
    "dram_bytes_write": ("dram__bytes_write.sum", 1, "byte"),
    "l2_bytes": ("lts__t_bytes.sum", 1, "byte"),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1, None),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1, None),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1, None),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1, None),
    "warp_exec_efficiency_threads": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1, None),
    "registers_per_thread": ("launch__registers_per_thread", 1, None),
    "l2_hit_rate_pct": ("lts__t_sector_hit_rate.pct", 1, None),
    "instructions": ("smsp__inst_executed.sum", 1, None),
    "grid": ("launch__grid_size", 1, None),
    "block": ("launch__block_size", 1, None),
}
UNIT = {"ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summary(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}
    d = {"kernel": vals[col["Kernel Name"]]}
    for key, (m, scale, base) in METRICS.items():
        if m not in col:
            continue
        v = float(vals[col[m]].replace(",", ""))
        u = units[col[m]]
        if base in ("ns",):
            v = v * UNIT.get(u, 1) * scale
        elif base == "byte":
            v = v * UNIT.get(u, 1)
        d[key] = round(v, 4) if isinstance(v, float) and not v.is_integer() else int(v)
    d["dram_bytes_per_launch"] = d.get("dram_bytes_read", 0) + d.get("dram_bytes_write", 0)
    stalls = {h[len("smsp__pcsamp_warps_issue_stalled_"):]: float(vals[i].replace(",", "") or 0)
              for h, i in col.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
    tot = sum(stalls.values()) or 1
    d["top_stalls_pct"] = {k: round(100 * v / tot, 1)
                           for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    return d


if __name__ == "__main__":
    print(json.dumps(summary(sys.argv[1]), indent=1))
