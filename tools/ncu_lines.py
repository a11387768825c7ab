"""Per-source-line stall samples from an ncu report (needs -lineinfo and
--import-source on): python tools/ncu_lines.py rep.ncu-rep [top]."""
import csv
import io
import subprocess
import sys


def main(path, top=40):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    fname, res, tot = "?", [], 0
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if len(r) < 8 or not r[0].isdigit() or r[2] != "-":
            continue
        s, inst = int(r[4] or 0), int(r[7] or 0)
        tot += s
        res.append((s, inst, f"{fname}:{r[0]}", r[1].strip()[:90]))
    res.sort(reverse=True)
    print(f"total samples {tot}")
    for s, inst, loc, src in res[:top]:
        print(f"{s:8d} {100.0 * s / max(tot, 1):5.1f}% {inst:12d}  {loc:24s} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
