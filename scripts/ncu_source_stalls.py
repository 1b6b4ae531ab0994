"""PC-sampling stalls per SASS instruction from an ncu capture made with
--set full --import-source on (run in the build container):

    python scripts/ncu_source_stalls.py REPORT.ncu-rep [kernel-regex] > profiles/<name>.txt

Per kernel: the stall-reason totals and the instructions with the most
samples (index in the kernel, samples, SASS, top reasons)."""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "Kernel Name":
        cur = {"name": row[1], "hdr": None, "rows": []}
        blocks.append(cur)
    elif cur is not None and cur["hdr"] is None:
        cur["hdr"] = row
    elif cur is not None:
        cur["rows"].append(row)
short = {"stall_long_sb": "long_sb", "stall_short_sb": "short_sb", "stall_math": "math", "stall_barrier": "barrier",
         "stall_wait": "wait", "stall_not_selected": "not_selected", "stall_selected": "selected",
         "stall_no_inst": "no_inst", "stall_dispatch": "dispatch", "stall_branch_resolving": "branch",
         "stall_lg": "lg_throttle", "stall_mio": "mio", "stall_membar": "membar", "stall_drain": "drain",
         "stall_sleeping": "sleeping", "stall_tex": "tex", "stall_imc": "imc_miss", "stall_misc": "misc"}
print(f"PC-sampling stalls per SASS instruction ({rep}; ncu --page source --print-source sass), top instructions by samples")
seen = set()
for b in blocks:
    if not re.search(kre, b["name"]) or b["name"] in seen:
        continue
    seen.add(b["name"])  # (one launch per kernel)
    h = b["hdr"]
    si = h.index("# Samples")
    cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    tot = {}
    rows = []
    for idx, r in enumerate(b["rows"]):
        s = int(r[si] or 0)
        rs = {short.get(n, n): int(r[i] or 0) for i, n in cols if int(r[i] or 0)}
        for k, v in rs.items():
            tot[k] = tot.get(k, 0) + v
        rows.append((s, idx, r[1].strip(), rs))
    n = sum(s for s, *_ in rows) or 1
    name = re.sub(r"\(int\)|\(bool\)|void mw::", "", b["name"]).split("(")[0]
    print(f"\n== {name}: {n} samples, {len(rows)} instructions")
    print("   totals: " + ", ".join(f"{k} {v} ({100 * v // n}%)" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:8]))
    for s, idx, sass, rs in sorted(rows, reverse=True)[:12]:
        top = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
        print(f"   # {idx:5d} {s:5d}  {sass[:48]:48s} {top}")
