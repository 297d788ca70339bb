"""Print ms/step and per-kernel ms for bench JSON lines given on the command line."""
import json
import sys

for f in sys.argv[1:]:
    try:
        d = json.loads([l for l in open(f) if l.startswith("{")][-1])
    except Exception as e:
        print(f, "no line", e)
        continue
    k = d["kernels"]
    def g(n, key="ms_per_launch"):
        return round(k.get(n, {}).get(key, float("nan")), 4)
    print(f"{f}: {d['ms_per_step']:.4f} ms/step  nb {g('nonbonded')}  list/rebuild {g('pairlist', 'ms_per_rebuild')}  "
          f"spread {g('spread')}  gather {g('gather')}  r2c {g('fft_r2c')}  lambda {g('lambda')}  e2e {d['e2e']['value']:.1f}")
