"""Writes profiles/README.md from the round's committed evidence files."""
import json, os, subprocess, sys
HERE = os.path.dirname(os.path.abspath(__file__))
D = os.path.join(os.path.dirname(HERE), "profiles")
table = subprocess.run([sys.executable, os.path.join(HERE, "profiles_table.py")], capture_output=True, text=True).stdout
b5 = json.load(open(os.path.join(D, "r01_bench_c5.json")))
b4 = json.load(open(os.path.join(D, "r01_bench_c4.json")))
c3 = json.load(open(os.path.join(D, "r01_c3_split.json")))
drift = [json.loads(l) for l in open(os.path.join(D, "r01_c5_power_drift.jsonl")) if l.strip()]
ro = b5.get("reordering", {})
e5 = b5["e2e"]
out = f"""# Round 1 measurements (B200, 1 GPU)

Bench lines: `r01_bench_c{{1..5}}.json` (`python bench.py --workload cN`; C5 is the default
workload).  SpMxV time = mean CUDA-event time of the apply calls in the timed region;
GB/s = algorithmic bytes (SURVEY §8(d)) / that time; frac = of the measured 6,534 GB/s copy
peak (MEASURED_PEAKS.json).  C1–C3 flush L2 (512 MB write) before every SpMxV (their warm-L2
time is listed too).  e2e = the step through the C ABI with x copied in and y copied out every
step (pinned host memory, copies pipelined against compute).  cuSPARSE = `cusparseSpMV` (via
`torch.mv` on an fp64 CSR tensor) on the same reordered matrix, same protocol, informational.

{table}
Second roofline of the panel kernel (`roofline_gather` in the C4/C5 lines): bytes crossing
L2 → SM per launch (group stream + the gathers' distinct 32-byte x sectors, counted at plan time)
over the SpMxV time, against a 128-bit LDG stream over an L2-resident buffer measured in the same
run: C5 {b5['roofline_gather']['bytes_per_launch'] / 1e9:.1f} GB per launch, {b5['roofline_gather']['achieved']:,.0f} of {b5['roofline_gather']['peak']:,.0f} GB/s =
**{b5['roofline_gather']['frac']:.2f}**; C4 {b4['roofline_gather']['bytes_per_launch'] / 1e9:.2f} GB, {b4['roofline_gather']['frac']:.2f}.  This fabric, not HBM, is what the C5
kernel runs into (DESIGN §5.1–5.2).

C5 and C4 time a power iteration (SpMxV with fused max-abs, max finish, x-update); the table's
SpMxV column is the SpMxV launch alone.  The C5 SpMxV runs under the board's power cap: a cold
GPU does it in {min(r['median_ms'] for r in drift[:1]):.2f} ms at {drift[0]['sm']} MHz, a warm one in
{drift[-1]['median_ms']:.2f} ms at {drift[-1]['sm']} MHz (`r01_c5_power_drift.jsonl`: 10 blocks of 20
back-to-back SpMxVs with the NVML clock, temperature, power and throttle reasons per block).

e2e (C5): {e5['value']:.1f} GFLOP/s, {e5['ms_per_step']:.2f} ms per step moving 512 MB in and 512 MB
out; the same copies alone take {e5.get('link_bound_ms_per_step', float('nan')):.2f} ms
({100 * e5.get('frac_of_link_bound', float('nan')):.0f} % of the e2e step): the host link bounds it.

Reordering effect (the paper's Table 2 analog, `reordering` in the C5 line): the same matrix in
its original scrambled order, row-tile kernel on the input CSR order {ro.get('scrambled_spmv_ms', float('nan')):.2f} ms
vs {ro.get('reordered_spmv_ms', float('nan')):.2f} ms SB-reordered: **{ro.get('speedup', float('nan')):.2f}×**; the panel
kernel on the scrambled matrix (its own column sort inside row panels recovers part of the
locality) {ro.get('scrambled_default_ms', float('nan')):.2f} ms.

C3 multiple-SpMxV (`r01_c3_split.json`, L2 flushed, SpMxV alone): single SpMxV
{c3['single_cold_ms']:.4f} ms, fused split on the panel kernel {c3['split_fused_cold_ms']:.4f} ms, literal K-pass
sequence {c3['split_literal_cold_ms']:.4f} ms ({c3['split_literal_cold_ms'] / c3['split_fused_cold_ms']:.1f}× the fused pass).

`roofline.traffic` in a bench line is read from `ncu_traffic.json` (DRAM bytes per launch of the
`--set full` capture of the same kernel, previous round-end run): C5 16.22 GB, C4 0.80 GB per
launch vs 14.72 / 0.66 GB algorithmic (group padding, per-group bases, the row→slot map and the x
prefetch).

Reproduce on a B200: `R=rNN bash scripts/final_round.sh` (GPU tests, smoke, the five bench lines,
the reference arm, the C3 split comparison, the power-drift trace, the C5 launch list and the
C5/C4 ncu captures, into `gpurun_out/`), then `python scripts/panel_md.py rNN` and
`python scripts/profiles_readme.py` after copying the lines here.  Interleaved A/B of plan or
library variants: `scripts/ab_inter.py`.

Kernel evidence: `r01_panel_c5_c4.md` (the C5 and C4 panel kernels, ncu `--set full`, per-SASS
memory counters), `r01_launches_c5.csv` (launch list of the C5 bench command), `r01_c5_rowtile.md`
(row-tile kernel on C5, earlier in the round), `r01_micro.json`, `r01_gather_modes.json`,
`r01_roofline_microbench.json`, `r01_diag_c5.json` (hardware bounds, DESIGN §5.1),
`ncu_traffic.json`.
"""
open(os.path.join(D, "README.md"), "w").write(out)
print(out)
