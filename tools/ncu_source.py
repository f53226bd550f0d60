"""Per-source-line hot spots of one kernel from an ncu --set full
--import-source capture: warp instructions executed and stall samples per
(file, line), largest first.

  python tools/ncu_source.py REPORT.ncu-rep KERNEL_REGEX [TOP]
"""
import csv
import io
import os
import subprocess
import sys


def rows(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kernel,
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    path = None
    header = None
    for rec in csv.reader(io.StringIO(out)):
        if not rec:
            continue
        if rec[0] == "File Path" or rec[0] == "File Name":
            path = rec[1]
            header = None
            continue
        if rec[0] == "Line No":
            header = rec
            continue
        if header and path and len(rec) > 3 and rec[2] == "-":  # per-CUDA-line aggregate
            d = dict(zip(header[4:], rec[4:]))
            d["Line No"], d["Source"] = rec[0], rec[1]
            yield path, d


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    agg = []
    tot_i = tot_s = 0
    for path, r in rows(rep, kernel):
        try:
            inst = float(r.get("Instructions Executed", "0") or 0)
            samp = float(r.get("Warp Stall Sampling (All Samples)", "0") or 0)
        except ValueError:
            continue
        if inst or samp:
            agg.append((inst, samp, os.path.basename(path), r["Line No"], r.get("Source", "")[:90]))
            tot_i += inst
            tot_s += samp
    agg.sort(reverse=True)
    print(f"total warp instructions {tot_i:.4g}, stall samples {tot_s:.4g}")
    for inst, samp, f, ln, src in agg[:top]:
        print(f"{100 * inst / tot_i:5.1f}% inst {100 * samp / max(tot_s, 1):5.1f}% stall  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()
