"""Per (stage, kind, kernel) sums of a bench --detail JSON's eager network launches."""
import json
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    d = json.load(open(path))
    agg = defaultdict(lambda: [0, 0.0])
    for l in d["network_launches"]:
        k = (l["stage"], l["kind"], l["name"])
        agg[k][0] += 1
        agg[k][1] += l["ms"]
    print(path, "forward", d["line"]["ms_per_step"], "dense", d["line"].get("dense_identity_ms_per_step"))
    for k in sorted(agg, key=lambda k: (str(k[0]), k[1], k[2])):
        n, ms = agg[k]
        print(f"  {str(k[0]):>4} {k[1]:>5} {k[2]:<16} n={n:3d} total {ms:7.3f} ms  mean {1e3 * ms / n:7.1f} us")
