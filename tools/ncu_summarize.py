#!/usr/bin/env python3
"""Summarise an `ncu --set full` capture of the iteration kernel into profiles/.

  python tools/ncu_summarize.py REPORT.ncu-rep TAG KEY K [--B 8192 --alg 443200 --eval 261600]

Writes profiles/<TAG>_details.csv (the details page), profiles/<TAG>_stalls.txt
(stall ratios, pipe / instruction counts) and records, under KEY (e.g.
"config4/F2") in profiles/ncu_summary.json, the DRAM bytes of the launch
against its algorithmic bytes  B*(K*alg + eval)  (K ascent iterations + the
final evaluation, which reads but does not write).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("tag")
    ap.add_argument("key")
    ap.add_argument("K", type=int)
    ap.add_argument("--B", type=int, default=8192)
    ap.add_argument("--alg", type=int, default=443200)
    ap.add_argument("--eval", dest="ev", type=int, default=261600)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    details = ncu(a.report, "--page", "details", "--csv")
    open(os.path.join(PROF, f"{a.tag}_details.csv"), "w").write(details)
    raw = list(csv.reader(io.StringIO(ncu(a.report, "--page", "raw", "--csv"))))
    h, u, v = raw[0], raw[1], raw[2]
    d = dict(zip(h, v))
    unit = dict(zip(h, u))

    def num(k):
        x = float(d[k].replace(",", ""))
        return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "Tbyte": 1e12}.get(unit[k], 1)

    lines = []
    for k in h:
        if ("issue_stalled" in k and k.endswith("per_issue_active.ratio")) or k.startswith("smsp__sass_inst_executed_op") \
                or k in ("smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                         "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
                         "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
            try:
                if float(d[k].replace(",", "")) != 0.0:
                    lines.append(f"{k} [{unit[k]}] = {d[k]}")
            except ValueError:
                pass
    open(os.path.join(PROF, f"{a.tag}_stalls.txt"), "w").write("\n".join(lines) + "\n")
    rd, wr = num("dram__bytes_read.sum"), num("dram__bytes_write.sum")
    alg = a.B * (a.K * a.alg + a.ev)
    ent = {"report": os.path.basename(a.report), "tag": a.tag, "launch_iterations": a.K,
           "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
           "alg_bytes_per_launch": alg, "dram_over_alg": round((rd + wr) / alg, 4),
           "gpu_time_ms": float(d["gpu__time_duration.sum"].replace(",", "")) *
           {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}[unit["gpu__time_duration.sum"]],
           "registers": d.get("launch__registers_per_thread"), "inst_executed": d.get("smsp__inst_executed.sum"),
           "note": a.note}
    path = os.path.join(PROF, "ncu_summary.json")
    js = json.load(open(path)) if os.path.exists(path) else {}
    js[a.key] = ent
    json.dump(js, open(path, "w"), indent=1)
    print(json.dumps(ent, indent=1))


if __name__ == "__main__":
    main()
