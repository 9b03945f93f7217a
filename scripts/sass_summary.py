"""Opcode summary of the engine's kernels from the built library (cuobjdump -sass): the tensor-core and
copy-engine instructions that prove the path (UTCHMMA / UTCQMMA = tcgen05.mma, UTMALDG = TMA tile load,
LDTM / STTM = TMEM load / store, HMMA = legacy mma.sync, LDSM = ldmatrix) and the total per kernel.

    python scripts/sass_summary.py > profiles/r02_sass_opcodes.txt
"""

import collections
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
LIB = ROOT / "paper_2001_06613_b200" / "libseqreg_b200.so"
WATCH = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UBLKCP", "LDTM", "STTM", "HMMA", "LDSM", "DFMA", "DADD",
         "F2F", "SHFL", "LDG", "STG", "LDS", "STS", "SYNCS"]
KEEP = ["k_ngf_sfeat2f", "k_gram_h", "k_ngf_z_tc", "k_ngf_adj4", "k_reduce_finalize", "k_sample_vp", "k_gram_tma",
        "k_pass2_tma", "k_pass2_mma", "k_ngf_z_f16", "k_ngf_feat4", "k_pass1_ws", "k_pass1<", "k_pass2<"]


def main():
    txt = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s+Function : ", txt)[1:]
    rows = []
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        short = dem.replace("void ", "").replace("sr::", "").split("(")[0]
        if not any(k.rstrip("<") in short for k in KEEP):
            continue
        ops = collections.Counter()
        for line in f.split("\n"):
            m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
            if m:
                ops[m.group(2)] += 1
        rows.append((short, sum(ops.values()), {k: ops[k] for k in WATCH if ops[k]}))
    print(f"cuobjdump -sass {LIB.name} (sm_100a): static instruction counts per kernel")
    seen = set()
    for short, tot, w in sorted(rows):
        key = (short, tot)
        if key in seen:  # (header-defined templates are instantiated in several translation units)
            continue
        seen.add(key)
        print(f"{short[:70]:70s} {tot:6d}  " + " ".join(f"{k}={v}" for k, v in w.items()))


if __name__ == "__main__":
    sys.exit(main())
