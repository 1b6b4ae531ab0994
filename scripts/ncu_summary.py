"""Summarise ncu captures into profiles/ (run in the build container).

    python scripts/ncu_summary.py ROUND report1.ncu-rep [report2 ...]

Writes profiles/<ROUND>_ncu_<kernel>.csv (the raw page, one row per launch)
and merges per-kernel key metrics into profiles/ncu_summary.json, which
bench.py reads for roofline.traffic (DRAM bytes per launch).
"""

import csv
import io
import json
import os
import re
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(REPO, "profiles")

KEYS = [
    "gpu__time_duration.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle",
    "smsp__pcsamp_warps_issue_stalled_wait",
    "smsp__pcsamp_warps_issue_stalled_barrier",
    "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_short_scoreboard",
    "smsp__pcsamp_warps_issue_stalled_not_selected",
    "smsp__pcsamp_warps_issue_stalled_selected",
]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def short(name):
    m = re.search(r"(\w+)<([^>]*)>", name)
    if m:
        return f"{m.group(1)}<{m.group(2).replace(' ', '')}>"
    return name.split("(")[0]


def main():
    rnd, reps = sys.argv[1], sys.argv[2:]
    os.makedirs(PROF, exist_ok=True)
    path = os.path.join(PROF, "ncu_summary.json")
    summary = json.load(open(path)) if os.path.exists(path) else {}
    for rep in reps:
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                             check=True).stdout
        rows = list(csv.reader(io.StringIO(raw)))
        hdr, units = rows[0], rows[1]
        for r in rows[2:]:
            kname = short(r[hdr.index("Kernel Name")])
            base = re.sub(r"[^A-Za-z0-9]+", "_", kname).strip("_")
            stem = os.path.splitext(os.path.basename(rep))[0]
            with open(os.path.join(PROF, f"{rnd}_ncu_{stem}_{base}.csv"), "w", newline="") as fh:
                w = csv.writer(fh)
                w.writerow(hdr)
                w.writerow(units)
                w.writerow(r)
            ent = {"round": rnd, "report": os.path.basename(rep)}
            for k in KEYS:
                if k in hdr:
                    i = hdr.index(k)
                    try:
                        v = float(r[i].replace(",", ""))
                    except ValueError:
                        continue
                    ent[k] = v * SCALE.get(units[i], 1) if units[i] in SCALE else v
                    ent[k + ".unit"] = "byte" if "byte" in units[i] else ("s" if "second" in units[i] else units[i])
            if "dram__bytes_read.sum" in ent and "dram__bytes_write.sum" in ent:
                ent["dram_bytes_per_launch"] = ent["dram__bytes_read.sum"] + ent["dram__bytes_write.sum"]
            prev = summary.get(kname)
            valid = "dram_bytes_per_launch" in ent and ent["dram_bytes_per_launch"] == ent["dram_bytes_per_launch"]
            if valid or prev is None:  # keep an earlier complete capture over a partial one
                summary[kname] = ent
            print(kname, json.dumps({k: v for k, v in ent.items() if not k.endswith(".unit")}, indent=None)[:400])
    json.dump(summary, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
