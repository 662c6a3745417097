"""Writes profiles/r01_panel_c5_c4.md from a round's ncu captures:
    python scripts/panel_md.py r98"""
import csv, json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, HERE)
import ncu_summary as N
R = sys.argv[1]
G = os.path.join(ROOT, "gpurun_out")
summ = lambda f: subprocess.run([sys.executable, os.path.join(HERE, "ncu_summary.py"), f], capture_output=True, text=True).stdout.strip()
S5, S4 = summ(os.path.join(G, f"{R}_panel_c5.ncu-rep")), summ(os.path.join(G, f"{R}_panel_c4.ncu-rep"))
T5, T4 = N.sass_table(os.path.join(G, f"{R}_panel_c5.ncu-rep")), N.sass_table(os.path.join(G, f"{R}_panel_c4.ncu-rep"))
rows = [r for r in csv.reader(open(os.path.join(ROOT, "profiles", "r01_launches_c5.csv"))) if len(r) > 5]
h = rows[0]
ik, iv, im = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = {}
for r in rows[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    k = r[ik].split("(")[0].replace("void ", "").replace("spmvb::<unnamed>::", "")
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r[iv].replace(",", ""))
tot = sum(v[1] for v in agg.values())
lt = "\n".join(f"| {k} | {v[0]} | {v[1] / 1e6:.3f} | {100 * v[1] / tot:.1f} % |" for k, v in sorted(agg.items(), key=lambda x: -x[1][1]))
b5 = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_c5.json")))
b4 = json.load(open(os.path.join(ROOT, "profiles", "r01_bench_c4.json")))
md = f"""# Round 1 — C5 (64M x 64M SB, 1.12e9 nnz) and C4 (4M x 4M power-law): the column-sorted panel kernel on B200

Commands (bench launch configuration): `python bench.py --workload c5|c4 --steps 3 --warmup 3 --no-e2e
--no-cpu-baseline --no-parity --no-gather-peak --no-reorder-ref --no-cusparse`; each ncu run wraps that command
right after it exited 0 without ncu (`scripts/final_round.sh`, gpurun_out/{R}_*).
Bench lines: `profiles/r01_bench_c5.json` — SpMxV {b5['spmv_ms']:.3f} ms = {b5['roofline']['achieved']:,.0f} GB/s
algorithmic = **{b5['roofline']['frac']:.3f} of the 6,534 GB/s measured copy peak** (clocks: {b5['clocks']});
`profiles/r01_bench_c4.json` — SpMxV {b4['spmv_ms']:.4f} ms, {b4['roofline']['frac']:.3f}.  The C5 SpMxV runs
power-capped after its first ≈ 0.1 s (`profiles/r01_c5_power_drift.jsonl`).

## Launch list (`profiles/r01_launches_c5.csv`, ncu `gpu__time_duration.sum`, cold-cache, serialised)

| kernel | launches | total ms | share |
|---|---|---|---|
{lt}

The SpMxV (with the fused max-abs) is {100 * max(v[1] for v in agg.values()) / tot:.1f} % of the power-iteration step;
the bench's live CUDA-event share agrees (SpMxV {b5['spmv_ms']:.3f} of {b5['ms_per_step']:.3f} ms per step).

## Full capture of the C5 kernel (`ncu --set full --clock-control none`, 1 launch)

{S5}

Per-instruction memory counters (source page), per executed warp instruction:

{T5}

Reading: `LDG.E.NA.64.CONSTANT` is the x gather (L1 no-allocate on SB handles) — ≈ 11.5 128-byte
lines and ≈ 22 sectors per 32 nonzeros (a row-ordered kernel: 32 lines); `LDG.E.NA.128.CONSTANT`
are the 16-byte stream loads (per warp and epoch two value pairs, one index quad, one base quad);
`LDS.64`/`STS.64` the shared-memory y read-modify-write (≈ 4 wavefronts each with the bank-coloured
slots, ideal 2).  L1TEX ≈ 89 % busy: its data stage and the L2→L1 fabric (the gathers re-read
each block's x(C_k) once per panel) bound the kernel, not HBM; DRAM traffic per launch ≈ 16.2 GB
vs 14.72 GB algorithmic (+10 %: group padding, per-group bases, the row→slot map, x prefetch).

## Full capture of the C4 kernel

{S4}

{T4}

Reading: C4's gather touches ≈ 10.4 lines per 32 nonzeros — its 30 % uniformly random columns,
one line and one sector each; neither L1TEX nor L2 saturates; the ablations (DESIGN §5.2) spread
the time over the gathers, the epoch barriers and the y updates.
"""
open(os.path.join(ROOT, "profiles", "r01_panel_c5_c4.md"), "w").write(md)
print(md[:1500])
