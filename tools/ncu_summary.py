"""Summarise an ncu --set full report (read here, after gpurun brought it back):
per kernel duration, DRAM bytes, instructions, issue activity, ALU/FMA pipe
utilisation and the top stall reasons -> JSON on stdout.

    python tools/ncu_summary.py gpurun_out/full_c1.ncu-rep [INPUT_BYTES] > profiles/rXX_ncu_full_c1.json

Values are in ncu's base units (bytes, ns; `units` lists them).  Also per
kernel: warp efficiency (active threads per executed warp instruction, of
32) and, given the parsed input's size, DRAM bytes per input byte.
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
    "smsp__thread_inst_executed_per_inst_executed.ratio",
]
STALLS = ["barrier", "branch_resolving", "dispatch_stall", "drain", "lg_throttle", "long_scoreboard",
          "math_pipe_throttle", "membar", "mio_throttle", "misc", "no_instruction", "not_selected", "selected",
          "short_scoreboard", "sleeping", "tex_throttle", "wait"]


def main(rep, input_bytes=None):
    names = METRICS + ["smsp__pcsamp_warps_issue_stalled_%s" % s for s in STALLS]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base",
                          "--metrics", ",".join(names)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))
    res = {"units": {m: units.get(m, "") for m in METRICS if units.get(m)}}
    if input_bytes:
        res["input_bytes"] = input_bytes
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
        try:
            e["warp_efficiency_pct"] = 100.0 * float(e["smsp__thread_inst_executed_per_inst_executed.ratio"]) / 32
            if input_bytes:
                e["dram_bytes_per_input_byte"] = (float(e["dram__bytes_read.sum"]) +
                                                  float(e["dram__bytes_write.sum"])) / input_bytes
        except (KeyError, ValueError):
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
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
