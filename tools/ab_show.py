"""Print value and per-kernel ms/step of tools/ab.sh outputs: python tools/ab_show.py PREFIX"""
import glob
import json
import sys

for f in sorted(glob.glob(f"gpurun_out/{sys.argv[1]}_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "FAILED", e)
        continue
    k = {n: round(v["ms_per_step"] * 1e3, 1) for n, v in d.get("kernels", {}).items()}
    print(f.split("_", 1)[1][:-5].ljust(14), round(d["value"], 1), k)
