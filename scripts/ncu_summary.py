"""Summarise an ncu report (--set full) into the numbers DESIGN.md and
bench.py's roofline use: duration, DRAM bytes per launch, L2/L1 hit rates,
throughputs, occupancy and the top warp-stall reasons.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [--json]
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex_evict_normal_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_evict_normal_lookup_miss.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "launch__grid_size",
    "launch__block_size",
    "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
]


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": v[hdr.index("Kernel Name")]}
        for i, h in enumerate(hdr):
            if h in KEYS:
                d[h] = (v[i], units[i])
        stalls = {}
        for i, h in enumerate(hdr):
            m = re.fullmatch(r"smsp__pcsamp_warps_issue_stalled_(\w+)", h)
            if m and not h.endswith("_not_issued"):
                try:
                    stalls[m.group(1)] = int(float(v[i]))
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        d["stalls_pct"] = {k: round(100.0 * c / tot, 1) for k, c in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
        res.append(d)
    return res


def to_bytes(val, unit):
    f = float(val)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    path = sys.argv[1]
    res = load(path)
    if "--json" in sys.argv:
        print(json.dumps(res, indent=1))
        return
    for d in res:
        print(f"### {d['kernel'][:100]}")
        t = d.get("gpu__time_duration.sum")
        rd = d.get("dram__bytes_read.sum")
        wr = d.get("dram__bytes_write.sum")
        if t and rd and wr:
            ms = float(t[0]) * {"ms": 1, "us": 1e-3, "ns": 1e-6, "s": 1e3}.get(t[1], 1)
            traffic = to_bytes(*rd) + to_bytes(*wr)
            print(f"- duration {ms:.4f} ms; DRAM traffic {traffic / 1e9:.3f} GB "
                  f"({traffic / (ms * 1e-3) / 1e9:.0f} GB/s under ncu, cold caches)")
        for k in KEYS[3:]:
            if k in d:
                print(f"- {k}: {d[k][0]} {d[k][1]}")
        print(f"- top stalls (% of samples): {d['stalls_pct']}")
        print()


if __name__ == "__main__":
    main()


def sass_table(path: str, min_exec: int = 1000000) -> str:
    """Per-SASS-opcode memory counters of the report's first kernel (source page),
    per executed warp instruction: L1 tag requests (global lines), shared
    wavefronts, L2 sectors."""
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    i_src, i_ex = h.index("Source"), h.index("Instructions Executed")
    cols = ["L1 Tag Requests Global", "L1 Wavefronts Shared", "L2 Theoretical Sectors Global"]
    ic = [h.index(c) for c in cols]
    agg = {}
    for r in rows[2:]:
        src = r[i_src].strip()
        op = src.split()[1] if src.startswith("@") else (src.split() or [""])[0]
        if not (op.startswith("LDG") or op.startswith("LDS") or op.startswith("STS") or op.startswith("STG")):
            continue
        ex = int(r[i_ex] or 0)
        a = agg.setdefault(op, [0, 0.0, 0.0, 0.0])
        a[0] += ex
        for j, i in enumerate(ic):
            a[j + 1] += float(r[i] or 0)
    lines = ["| SASS | executed | L1 tag requests (global lines) | shared wavefronts | L2 sectors |", "|---|---|---|---|---|"]
    for op, a in agg.items():
        if a[0] >= min_exec:
            lines.append(f"| {op} | {a[0]} | {a[1] / a[0]:.2f} | {a[2] / a[0]:.2f} | {a[3] / a[0]:.2f} |")
    return "\n".join(lines)
