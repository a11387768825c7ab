#!/bin/bash
# Copy tools/ncu_all.sh results from gpurun_out/ into profiles/ (tracked).
set -eu
tag=$1
mkdir -p profiles/$tag
cp gpurun_out/ncu_$tag/march_*_ncu.txt profiles/$tag/
python - "$tag" <<'PY'
import json, os, sys
tag = sys.argv[1]
src = f"gpurun_out/ncu_{tag}/ncu_counters.json"
dst = "profiles/ncu_counters.json"
new = json.load(open(src))
doc = json.load(open(dst)) if os.path.exists(dst) else {}
doc.update(new)
json.dump(doc, open(dst, "w"), indent=1, sort_keys=True)
print("updated", dst, sorted(k for k in new if not k.startswith("_")))
PY
