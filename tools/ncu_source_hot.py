"""Top SASS hot spots (warp stall samples) of one kernel in an ncu report (--import-source capture).
  python tools/ncu_source_hot.py gpurun_out/prof.ncu-rep "<substring of kernel name>" [top] [occurrence]"""
import csv, io, subprocess, sys

rep, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
occ = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                              text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(out)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif cur is not None:
        cur["rows"].append(r)
sel = [b for b in blocks if pat in b["name"].replace("(int)", "").replace("(bool)", "")]
if not sel:
    print("kernels:", [b["name"] for b in blocks])
    sys.exit(1)
b = sel[min(occ, len(sel) - 1)]
hdr = b["rows"][0]
src_c = hdr.index("Source")
samp_c = hdr.index("Warp Stall Sampling (All Samples)")
recs = []
for r in b["rows"][1:]:
    try:
        recs.append((float(r[samp_c]), r[src_c]))
    except (ValueError, IndexError):
        pass
tot = sum(v for v, _ in recs) or 1
print(b["name"], f"samples {tot:.0f} instructions {len(recs)}")
by_op = {}
for v, s in recs:
    t = s.strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    by_op[op.split(".")[0]] = by_op.get(op.split(".")[0], 0) + v
print(" by opcode:", ", ".join(f"{op} {v / tot:.3f}" for op, v in sorted(by_op.items(), key=lambda kv: -kv[1])[:14]))
for v, s in sorted(recs, reverse=True)[:top]:
    print(f"{v / tot:6.3f}  {s.strip()[:90]}")
