"""Summarise an ncu --set full report (read here, after gpurun brought it back):
per kernel duration, DRAM bytes, instructions, issue activity, ALU/FMA pipe
utilisation and the top stall reasons -> JSON on stdout.

    python tools/ncu_summary.py gpurun_out/full_c1.ncu-rep > profiles/rXX_ncu_full_c1.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
]
STALLS = ["barrier", "branch_resolving", "dispatch_stall", "drain", "lg_throttle", "long_scoreboard",
          "math_pipe_throttle", "membar", "mio_throttle", "misc", "no_instruction", "not_selected", "selected",
          "short_scoreboard", "sleeping", "tex_throttle", "wait"]


def main(rep):
    names = METRICS + ["smsp__pcsamp_warps_issue_stalled_%s" % s for s in STALLS]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(names)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        k = d["Kernel Name"].split("(")[0].replace("void ", "").replace("jt::<unnamed>::", "").replace("jt::", "")
        e = {m: d.get(m) for m in METRICS if d.get(m) not in (None, "", "n/a")}
        st = {}
        for s in STALLS:
            v = d.get("smsp__pcsamp_warps_issue_stalled_%s" % s)
            try:
                st[s] = float(v)
            except (TypeError, ValueError):
                pass
        tot = sum(st.values()) or 1.0
        e["top_stalls"] = ", ".join("%s %d%%" % (s, round(100 * v / tot)) for s, v in
                                    sorted(st.items(), key=lambda kv: -kv[1])[:4])
        key = k
        i = 2
        while key in res:
            key = "%s#%d" % (k, i)
            i += 1
        res[key] = e
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
