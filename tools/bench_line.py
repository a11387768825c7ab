"""Print the key fields of the bench JSON line(s) in a file: tools/bench_line.py [FILE|-] [label]."""
import json
import sys

label = sys.argv[2] if len(sys.argv) > 2 else ""
for line in (open(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1] != "-" else sys.stdin):
    line = line.strip()
    if not line.startswith("{"):
        continue
    try:
        d = json.loads(line)
    except ValueError:
        continue
    r = d.get("roofline", {})
    print(label, d.get("config", {}).get("workload", "")[:4], "fps", d.get("value"), "Gs/s", d.get("gsamples_per_s"),
          "frac", r.get("frac"), "kernel_ms", r.get("kernel_ms"), "e2e", (d.get("e2e") or {}).get("value"))
