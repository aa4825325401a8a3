"""Per-source-line summary of an ncu report's source page (stall samples and
executed instructions), from `ncu -i X --page source --csv --print-source sass,cuda`.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    lines = []
    for r in rows:
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and r and r[0].isdigit() and len(r) > 8 and r[2] == "-":
            d = dict(zip(hdr[2:], r[2:]))
            try:
                samp = int(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
                inst = int(d.get("Instructions Executed", 0) or 0)
            except ValueError:
                continue
            lines.append((samp, inst, int(r[0]), r[1].strip()[:90]))
    tot_s = sum(l[0] for l in lines) or 1
    tot_i = sum(l[1] for l in lines) or 1
    print(f"total samples {tot_s}, warp instructions {tot_i}")
    for samp, inst, ln, src in sorted(lines, reverse=True)[:top]:
        print(f"{100 * samp / tot_s:5.1f}% samp {100 * inst / tot_i:5.1f}% inst  L{ln:4d}  {src}")


if __name__ == "__main__":
    main()
