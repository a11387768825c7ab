#!/bin/bash
# One `ncu --set full` capture of the dominant march kernel per bench config
# (C1-C5 single camera, C4 3-point TF), summaries into profiles/$1/ and the
# counters into profiles/ncu_counters.json.   usage: tools/ncu_all.sh r2
set -u
tag=$1
mkdir -p profiles/$tag gpurun_out
for c in c4 c2 c3 c1 c5; do
  ncu --set full --import-source on --clock-control none -k regex:march -c 1 -f -o gpurun_out/${tag}_$c \
      python tools/time_march.py --config $c --reps 1 > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/${tag}_$c.ncu-rep > profiles/$tag/march_${c}_ncu.txt
  python tools/ncu_lines.py gpurun_out/${tag}_$c.ncu-rep 30 >> profiles/$tag/march_${c}_ncu.txt
  python tools/ncu_counters.py ${c}_n1 gpurun_out/${tag}_$c.ncu-rep profiles/$tag/march_${c}_ncu.txt
done
