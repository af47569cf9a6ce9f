"""One line per config of a bench.py JSON line (all_configs)."""
import json
import sys

d = json.loads([ln for ln in open(sys.argv[1]) if ln.startswith("{")][-1])
print("headline", d["config"]["workload"], f"{d['value']:.4g}", d["unit"],
      f"ms/step {d['ms_per_step']:.4f}", "clocks", d.get("clocks"))
for k, r in d.get("all_configs", {}).items():
    ip = r.get("int_pipe", {})
    print(k, f"ms {r.get('ms_per_step', 0):.4f}", f"value {r['value']:.4g}",
          f"hbm {r.get('roofline', {}).get('frac', 0):.3f}",
          f"int_nom {ip.get('frac', 0):.3f} int_prac {ip.get('practical_frac', 0):.3f}",
          f"e2e {r.get('e2e', {}).get('value', 0):.4g}",
          f"cpu {r.get('cpu_baseline', {}).get('value', 0):.4g}",
          f"launches {r.get('gpu_launches')}", r.get("launch"))
