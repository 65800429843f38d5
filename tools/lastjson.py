"""Print selected keys of the last JSON line of a bench output file (development helper)."""
import json
import sys

for path in sys.argv[1:]:
    try:
        line = [l for l in open(path) if l.startswith("{")][-1]
        d = json.loads(line)
    except Exception as e:
        print(path, "no json:", e)
        continue
    keys = ["us_per_layer_step", "stages_us", "phases_us_per_layer", "speedup_vs_dense"]
    print(path, {k: (round(d[k], 2) if isinstance(d.get(k), float) else d.get(k)) for k in keys if k in d})
