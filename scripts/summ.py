import json, sys
for f in sys.argv[1:]:
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "ERR", open(f).read()[-2000:]); continue
    r = d.get("roofline", {})
    print(f.split('/')[-1], f"{d['value']:.4g}", d['unit'], "kernel_ms", round(r.get('kernel_ms', 0), 4),
          "frac", round(r.get('frac', 0), 4), "e2e", f"{(d.get('e2e') or {}).get('value', 0):.4g}",
          "int_frac", round(d.get('int_pipe', {}).get('frac', 0), 3), "clk", d.get('clocks', {}).get('sm_mhz'),
          d.get('clocks', {}).get('reasons'))
