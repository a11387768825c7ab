#!/bin/bash
# One `ncu --set full` capture of the dominant march kernel per bench config
# (C1-C5, single camera).  Writes the reports and the per-config summaries
# under gpurun_out/ (the only directory gpurun brings back), and the
# counters file gpurun_out/ncu_counters.json; copy the summaries to
# profiles/$tag/ and the counters to profiles/ncu_counters.json afterwards
# (tools/ncu_import.sh).   usage: tools/ncu_all.sh r2 [configs...]
# A config "cNlut" captures config cN with the shared-memory LUT forced
# (the bench line's lut_path block reads it as cN_lut_n1), "cNet" with early
# termination at alpha_stop 0.99 and the TF opacity x0.01 (early_termination
# block, cN_et_n1), "cNtf4" with bench.py's 4-point transfer function
# (tf_4point block, cN_tf4_n1).
TF4='[[0,0,0,0,0],[0.21,0.5,0.1,0.1,0.05],[0.63,0.1,0.9,0.3,0.4],[1,1,1,1,0.9]]'
set -u
tag=$1; shift
cfgs=${*:-c4 c2 c3 c1 c5}
out=gpurun_out/ncu_$tag
mkdir -p $out
for c in $cfgs; do
  # C3 renders in two passes (iso probe + volume march): capture both
  n=1; [ "$c" = c3 ] && n=2
  base=$c; extra=(); key=${c}_n1
  case $c in
    *lut) base=${c%lut}; extra=(--lut); key=${base}_lut_n1 ;;
    *et)  base=${c%et}; extra=(--alpha 0.99 --opacity 0.01); key=${base}_et_n1 ;;
    *tf4) base=${c%tf4}; extra=(--points "$TF4"); key=${base}_tf4_n1 ;;
  esac
  ncu --set full --import-source on --clock-control none -k regex:"march|iso_probe" -c $n -f -o $out/$c \
      python tools/time_march.py --config $base --reps 1 "${extra[@]}" > /dev/null 2>&1
  python tools/ncu_summary.py $out/$c.ncu-rep > $out/march_${c}_ncu.txt
  python tools/ncu_lines.py $out/$c.ncu-rep 30 >> $out/march_${c}_ncu.txt
  if [ "$c" = c3 ]; then
    NCU_COUNTERS=$out/ncu_counters.json python tools/ncu_counters.py c3_n1 $out/$c.ncu-rep profiles/$tag/march_c3_ncu.txt march_fast_kernel
    NCU_COUNTERS=$out/ncu_counters.json python tools/ncu_counters.py c3_probe_n1 $out/$c.ncu-rep profiles/$tag/march_c3_ncu.txt iso_probe
  else
    NCU_COUNTERS=$out/ncu_counters.json python tools/ncu_counters.py $key $out/$c.ncu-rep profiles/$tag/march_${c}_ncu.txt
  fi
  # reports are large; gpurun brings back at most 64 MiB of gpurun_out/
  if [ -z "${NCU_KEEP:-}" ]; then rm -f "gpurun_out/ncu_${tag}/${c}.ncu-rep"; fi
done
