#!/usr/bin/env python3
"""Summarise the PTDF dense-path profiles (tools/gpu_ptdf_ncu.sh) into profiles/:
the launch list (per-launch time and DRAM bytes of GEMM1 / GEMM2 / finisher),
the ncu --set full details page of the two fused GEMMs, their stall breakdown by
SASS opcode, and an entry "config4b/PTDF" in profiles/ncu_summary.json with the
per-launch fp64 rate (algorithmic flops 2 n_l n_g B per GEMM / ncu time)."""
import csv
import io
import json
import os
import shutil
import subprocess
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")
SRC = os.path.join(ROOT, "gpurun_out", "ptdf")
NL, NG, B = 12700, 2500, 8192
CHUNKS = 2  # iterate() runs the batch as two column groups on two streams: one launch covers B / 2


def main():
    shutil.copy(os.path.join(SRC, "launches.csv"), os.path.join(PROF, "r1_ptdf_launches_config4b.csv"))
    rows = list(csv.reader(open(os.path.join(SRC, "launches.csv"))))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[start]
    ix = {k: j for j, k in enumerate(h)}
    per = {}
    for r in rows[start + 1:]:
        if len(r) < len(h):
            continue
        per.setdefault((int(r[ix["ID"]]), r[ix["Kernel Name"]]), {})[r[ix["Metric Name"]]] = float(
            r[ix["Metric Value"]].replace(",", ""))
    kinds = {"k_dgemm<1>": "GEMM1 (gen epilogue)", "k_dgemm<2>": "GEMM2 (line epilogue, step)",
             "k_finish<0>": "finisher"}
    agg = {}
    for (i, name), m in sorted(per.items()):
        for key, label in kinds.items():
            if key in name.replace("(int)", ""):
                agg.setdefault(label, []).append(m)
    out = {}
    for label, ms in agg.items():
        t = sum(x["gpu__time_duration.sum"] for x in ms) / len(ms) / 1e6
        rd = sum(x["dram__bytes_read.sum"] for x in ms) / len(ms)
        wr = sum(x["dram__bytes_write.sum"] for x in ms) / len(ms)
        e = {"launches": len(ms), "gpu_time_ms": round(t, 4), "dram_read": rd, "dram_write": wr}
        if "GEMM" in label:
            e["fp64_tflops"] = round(2.0 * NL * NG * (B / CHUNKS) / (t / 1e3) / 1e12, 2)
        out[label] = e
    rep = os.path.join(SRC, "ncu_dgemm.ncu-rep")
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    open(os.path.join(PROF, "r1_ptdf_ncu_dgemm_details.csv"), "w").write(det)
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    lines, blocks, cur = src.split("\n"), [], None
    for ln in lines:
        if ln.startswith('"Kernel Name"'):
            cur = [ln]
            blocks.append(cur)
        elif cur is not None:
            cur.append(ln)
    txt = []
    for b in blocks:
        rs = list(csv.reader(b[1:]))
        hh = rs[0]
        j = {k: i for i, k in enumerate(hh)}
        data = [r for r in rs[1:] if len(r) == len(hh)]
        tot = sum(int(r[j["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
        txt.append(f"{b[0][:90]}  samples={tot}")
        for key in ["stall_wait", "stall_math", "stall_long_sb", "stall_short_sb", "stall_barrier", "stall_selected",
                    "stall_not_selected", "stall_dispatch", "stall_mio"]:
            cc = Counter()
            for r in data:
                op = r[j["Source"]].split()
                if not op:
                    continue
                o = op[1] if op[0].startswith("@") else op[0]
                cc[o.split(".")[0]] += int(r[j[key]] or 0)
            s = sum(cc.values())
            txt.append(f"  {key:20s} {s:8d} ({100.0 * s / max(tot, 1):5.1f}%)  top: {cc.most_common(3)}")
    open(os.path.join(PROF, "r1_ptdf_ncu_dgemm_stalls.txt"), "w").write(
        "ncu --set full of k_dgemm<2> (GEMM2) and k_dgemm<1> (GEMM1), config 4b PTDF, 64x128x16 tiles, 2 CTAs/SM.\n"
        "stall_wait / stall_math on DMMA and the NOPs ptxas pairs with each DMMA = the DMMA pipe saturated.\n"
        + "\n".join(txt) + "\n")
    summ = json.load(open(os.path.join(PROF, "ncu_summary.json")))
    summ["config4b/PTDF"] = {"per_kernel": out, "tag": "r1_ptdf_ncu_dgemm",
                             "alg_flops_per_gemm_launch": 2 * NL * NG * B // CHUNKS,
                             "note": "ncu launch list (serialised, cold) of bench.py --workload config4b --form PTDF; "
                                     "the bench line's rate is the whole step over CUDA events"}
    json.dump(summ, open(os.path.join(PROF, "ncu_summary.json"), "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
