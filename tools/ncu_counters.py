"""Record the dominant kernel's ncu counters per bench config into
profiles/ncu_counters.json (read by bench.py for roofline.traffic and
roofline.l1tex):

    python tools/ncu_counters.py c4_n1 gpurun_out/c4.ncu-rep profiles/r2/march_c4_ncu.txt [kernel-substring]

The report is one `ncu --set full --clock-control none` capture of the
kernel (e.g. of `python tools/time_march.py --config c4 --reps 1`)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("NCU_COUNTERS") or os.path.join(ROOT, "profiles", "ncu_counters.json")
METRICS = {
    "dram__bytes_read.sum": "dram_read_bytes",
    "dram__bytes_write.sum": "dram_write_bytes",
    "gpu__time_duration.sum": "duration",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed": "l1tex_data_pipe_lsu_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "l1tex__t_sector_hit_rate.pct": "l1_hit_rate_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers_per_thread",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def read(rep, kernel=""):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")]
        if kernel and kernel not in name:
            continue
        res = {"kernel": name}
        for m, key in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if key.endswith("_bytes"):
                v *= SCALE.get(u, 1)
            if key == "duration":
                key, v = "duration_ms", v * SCALE.get(u, 1)
            res[key] = v
        return res
    raise SystemExit(f"no kernel matching {kernel!r} in {rep}")


def main():
    key, rep, summary = sys.argv[1:4]
    kernel = sys.argv[4] if len(sys.argv) > 4 else "march"
    res = read(rep, kernel)
    res["traffic_bytes"] = int(res.pop("dram_read_bytes", 0) + res.pop("dram_write_bytes", 0))
    res["source"] = summary
    doc = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            doc = json.load(fh)
    doc["_doc"] = ("dominant-kernel counters per bench config from one `ncu --set full --clock-control none` "
                   "capture each (tools/ncu_counters.py); traffic_bytes = dram__bytes_read.sum + "
                   "dram__bytes_write.sum per launch; l1tex_data_pipe_lsu_pct = "
                   "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed (the march's real limiter)")
    doc[key] = res
    with open(OUT, "w") as fh:
        json.dump(doc, fh, indent=1, sort_keys=True)
    print(json.dumps({key: res}))


if __name__ == "__main__":
    main()
