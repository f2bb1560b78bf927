"""Markdown table of a bench.py line (headline + every config under "configs")."""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
rows = [(d["config"]["workload"].split(":")[0], d)] + list(d.get("configs", {}).items())
print("| config | solves/s | ms/step | stages ms (detect / factor+rcond+solve / take or fallback) | roofline | e2e solves/s | CPU oracle solves/s |")
print("|---|---|---|---|---|---|---|")
for tag, c in rows:
    r = c.get("roofline", {})
    st = r.get("stage_ms") or []
    roof = f"{r.get('bound')} {100 * r.get('frac', 0):.2f}% ({r.get('achieved', 0):.3g} {r.get('unit', '')})"
    dk = r.get("dominant_kernel")
    if dk:
        roof += f"; kernel {dk['name']} {100 * dk['frac']:.1f}%"
    print(f"| {tag} | {c['value']:.4g} | {c['ms_per_step']:.4g} | {' / '.join(f'{x:.3g}' for x in st[:3])} | {roof} | "
          f"{c.get('e2e', {}).get('value', 0):.4g} | {c.get('cpu_baseline', {}).get('value', 0):.3g} |")
