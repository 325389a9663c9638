"""Summarise an `ncu --set full` capture of the K1 kernels into
profiles/k1_ncu_summary.json (read by bench.py for roofline.traffic and the
issue-rate figure).

  ncu -i rep --page raw --csv > raw.csv
  python tools/ncu_summary.py raw.csv --dags 1000000 --div-groups-per-dag 14.54 --out profiles/k1_ncu_summary.json
"""
import argparse
import csv
import json
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("raw")
    ap.add_argument("--dags", type=int, default=1000000)
    ap.add_argument("--div-groups-per-dag", type=float, required=True)
    ap.add_argument("--command", default="")
    ap.add_argument("--version", default="")
    ap.add_argument("--out", required=True)
    ap.add_argument("--details", default="", help="ncu --page details --csv of the same report (active threads/warp)")
    a = ap.parse_args()
    rows = list(csv.reader(open(a.raw)))
    h, units = rows[0], rows[1]
    col = {k: i for i, k in enumerate(h)}

    def val(r, k):
        i = col[k]
        x = float(r[i].replace(",", "") or 0)
        u = units[i]
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "ms": 1e-3, "us": 1e-6, "ns": 1e-9,
                 "msecond": 1e-3, "usecond": 1e-6, "nsecond": 1e-9, "MHz": 1e6, "GHz": 1e9, "Mhz": 1e6, "Ghz": 1e9}.get(u, 1)
        return x * scale

    out = {"round": 2, "version": a.version, "command": a.command, "dags": a.dags,
           "division_groups_per_dag": a.div_groups_per_dag, "kernels": {}}
    for r in rows[2:]:
        name = re.sub(r"^void ", "", r[col["Kernel Name"]])
        name = re.sub(r"\(.*", "", name).replace("ds::", "")
        if not name.startswith("k1_fast"):  # bench.py names k1_fast<32>/<64> by slot count, the rest bare
            name = re.sub(r"<.*", "", name)
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): val(r, k) for k in h
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        tot = sum(stalls.values()) or 1.0
        top = dict(sorted(((k, round(100 * v / tot, 1)) for k, v in stalls.items()), key=lambda t: -t[1])[:6])
        d = {"duration_ms": val(r, "gpu__time_duration.sum") * 1e3,
             "dram_bytes_read": val(r, "dram__bytes_read.sum"),
             "dram_bytes_write": val(r, "dram__bytes_write.sum"),
             "warp_instructions": val(r, "smsp__inst_executed.sum"),
             "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
             "warps_active_per_sm": val(r, "sm__warps_active.avg.per_cycle_active"),
             "registers_per_thread": val(r, "launch__registers_per_thread"),
             "top_stalls_pct": top}
        for k in ("smsp__thread_inst_executed.sum", "smsp__thread_inst_executed_pred_on.sum"):
            if k in col and d["warp_instructions"]:
                d["threads_per_warp_instr" if k.endswith("executed.sum") else "pred_on_threads_per_warp_instr"] = \
                    val(r, k) / d["warp_instructions"]
        d["dram_bytes_per_dag"] = (d["dram_bytes_read"] + d["dram_bytes_write"]) / a.dags
        d["warp_instructions_per_dag"] = d["warp_instructions"] / a.dags
        out["kernels"][name] = d
        out["sm_count"] = int(val(r, "device__attribute_multiprocessor_count")) if "device__attribute_multiprocessor_count" in col else 148
        if "sm__cycles_elapsed.avg.per_second" in col and "sm_clock_mhz" not in out:
            out["sm_clock_mhz"] = val(r, "sm__cycles_elapsed.avg.per_second") / 1e6
    if a.details:
        for r in csv.reader(open(a.details)):
            if len(r) > 14 and r[12] in ("Avg. Active Threads Per Warp", "Avg. Not Predicated Off Threads Per Warp"):
                name = re.sub(r"\(.*", "", re.sub(r"^void ", "", r[4]))
                if not name.startswith("k1_fast"):
                    name = re.sub(r"<.*", "", name)
                key = "threads_per_warp_instr" if "Active" in r[12] else "pred_on_threads_per_warp_instr"
                if name in out["kernels"]:
                    out["kernels"][name][key] = float(r[14])
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
