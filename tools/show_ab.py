import json, sys
for l in open(sys.argv[1]):
    if l.startswith('=='): print(l.strip()); continue
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print(f"  {d['config']} n={d['n']} B={d['B']} kernel={d['kernel_us']:.2f}us step={d['step_us']:.2f}us frac={d['frac']:.3f}")
