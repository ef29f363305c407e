"""SASS evidence for profiles/: the instruction mix of the product kernels a C2 KeySwitch launches, read from
the built libhks.so with cuobjdump (here, on the CPU box).  It shows which pipe each kernel's arithmetic lands
on: tcgen05 (UTCIMMA = tcgen05.mma, LDTM = tcgen05.ld), TMA / bulk copies (UTMALDG, UBLKCP), cp.async
(LDGSTS), and the integer multiplies of the Shoup / 30-bit-split arithmetic on the FMA-heavy pipe
(IMAD.WIDE, IMAD.HI, IMAD, IMAD.X).

  python tools/sass_summary.py --name r4 [--so paper_2507_04775_b200/libhks.so]  -> profiles/sass_<name>.md
"""
import argparse
import collections
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# the kernels of one C2 KeySwitch (launch order) and what they compute
KERNELS = [
    ("_Z5k_nttILi8ELi3ELi3ELi8ELb0ELb0ELi0EEv7NttArgs", "ntt_inv_rows", "INTT row pass of c1 (GS, radix-8)"),
    ("_Z5k_nttILi8ELi4ELi3ELi8ELb1ELb0ELi3EEv7NttArgs", "ntt_inv_cols_scale", "INTT column pass + Eq. 1 / ModDown scale"),
    ("_Z10k_bconv_tcILi10ELb1EEv9BconvArgs", "bconv", "ModUp / ModDown base conversion (Eq. 1) on tcgen05"),
    ("_Z5k_nttILi8ELi4ELi4ELi8ELb1ELb1ELi0EEv7NttArgs", "ntt_fwd_cols", "NTT column pass, 90-limb batch (CT, radix-16)"),
    ("_Z9k_ntt_kipILi8ELi4ELi2ELi3ELi3EEv12FusedKipArgs", "ntt_rows_kip", "NTT row pass + key inner product + ModDown INTT rows"),
    ("_Z5k_nttILi8ELi3ELi3ELi8ELb0ELb1ELi2EEv7NttArgs", "ntt_fwd_rows_moddown", "NTT row pass + (acc - x) P^-1 + c0 epilogue"),
]
OPS = ["UTCIMMA", "LDTM", "UTMALDG", "UBLKCP", "LDGSTS", "IMAD.WIDE.U32", "IMAD.HI.U32", "IMAD", "IMAD.X",
       "IMAD.MOV.U32", "IADD3", "IADD3.X", "LDG", "STG", "LDS", "STS", "BAR", "SYNCS"]


EXACT = {"IMAD.WIDE.U32", "IMAD.HI.U32", "IMAD", "IMAD.X", "IMAD.MOV.U32", "IADD3", "IADD3.X"}


def opcode_counts(so, fn):
    out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, so], capture_output=True, text=True).stdout
    c = collections.Counter()
    total = 0
    for line in out.splitlines():
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[0-9T]+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        op = m.group(1)
        total += 1
        if op in EXACT:
            c[op] += 1
        else:
            base = op.split(".")[0]
            if base in OPS:
                c[base] += 1
    return total, c


def ptxas_info(fn):
    """registers / spills from the build logs (paper_2507_04775_b200/build/*.o.log, -Xptxas -v)"""
    logdir = os.path.join(ROOT, "paper_2507_04775_b200", "build")
    for f in sorted(os.listdir(logdir)) if os.path.isdir(logdir) else []:
        if not f.endswith(".log"):
            continue
        lines = open(os.path.join(logdir, f)).read().splitlines()
        for i, l in enumerate(lines):
            if f"Compiling entry function '{fn}'" in l:
                spill = regs = ""
                for l2 in lines[i + 1:i + 6]:
                    m = re.search(r"(\d+) bytes spill stores", l2)
                    if m:
                        spill = m.group(1)
                    m = re.search(r"Used (\d+) registers", l2)
                    if m:
                        regs = m.group(1)
                        break
                return regs, spill
    return "", ""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--name", required=True)
    ap.add_argument("--so", default=os.path.join(ROOT, "paper_2507_04775_b200", "libhks.so"))
    a = ap.parse_args()
    rows = []
    for fn, cls, what in KERNELS:
        total, c = opcode_counts(a.so, fn)
        regs, spill = ptxas_info(fn)
        rows.append((cls, what, fn, total, c, regs, spill))
    path = os.path.join(ROOT, "profiles", f"sass_{a.name}.md")
    with open(path, "w") as f:
        f.write(f"# SASS instruction mix: {a.name}\n\n")
        f.write("`cuobjdump -sass` of the built `libhks.so` (sm_100a), static instruction counts per kernel "
                "(`tools/sass_summary.py`). UTCIMMA = `tcgen05.mma`, LDTM = `tcgen05.ld`, UBLKCP = bulk copy, "
                "UTMALDG = TMA tensor load, LDGSTS = `cp.async`; IMAD.WIDE / IMAD.HI / IMAD / IMAD.X issue on the "
                "FMA-heavy pipe. Registers and spill bytes from `ptxas -v`.\n\n")
        f.write("| class | kernel | SASS | regs | spill B | " + " | ".join(k for k in OPS) + " |\n")
        f.write("|---|---|---|---|---|" + "---|" * len(OPS) + "\n")
        for cls, what, fn, total, c, regs, spill in rows:
            f.write(f"| {cls} | {what} | {total} | {regs} | {spill} | " + " | ".join(str(c.get(k, 0)) for k in OPS) + " |\n")
    print(path)


if __name__ == "__main__":
    main()
