"""Prints the profiles/README.md summary table from profiles/r01_bench_c*.json."""
import json, os
D = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
print("| cfg | SpMxV ms | GB/s (alg) | frac | GFLOP/s (step) | e2e GFLOP/s | warm-L2 ms | cuSPARSE ms (ours ×) "
      "| kernel | parity (sampled rows) | oracle GFLOP/s (host cores) |")
print("|---|---|---|---|---|---|---|---|---|---|---|")
for c in ("c1", "c2", "c3", "c4", "c5"):
    j = json.load(open(os.path.join(D, f"r01_bench_{c}.json")))
    r = j["roofline"]
    cs = j.get("cusparse", {})
    par = j.get("parity", {})
    cpu = j.get("cpu_baseline", {})
    warm = j.get("warm_l2_spmv_ms")
    print(f"| {c.upper()} | {j['spmv_ms']:.4f} | {r['achieved']:,.0f} | {r['frac']:.3f} | {j['value']:.1f} "
          f"| {j['e2e']['value']:.1f} | {'' if warm is None else f'{warm:.4f}'} "
          f"| {cs.get('spmv_ms', float('nan')):.4f} ({cs.get('speedup_ours', float('nan')):.2f}×) "
          f"| {j['config']['kernel']} | {par.get('failures', '?')} failures / {par.get('rows_checked', '?')} "
          f"| {cpu.get('value', float('nan')):.2f} ({cpu.get('cores', '?')} cores) |")
