import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline") or {}
    print(f"{f}: value={d['value']:.4g} e2e={d['e2e']['value']:.4g} seeded={d.get('e2e_seeded',{}).get('value',0):.4g} "
          f"ms/step={d['ms_per_step']:.4f} launches={d.get('gpu_launches')} stages={ {k: round(v*1e3,1) for k,v in (d.get('stage_ms_per_round') or {}).items()} } "
          f"roof={r.get('kernel')} {r.get('achieved',0):.4g}/{r.get('peak')} frac={r.get('frac',0):.4g} cpu={(d.get('cpu_baseline') or {}).get('value')} clocks={d.get('clocks',{}).get('sm_mhz')}")
