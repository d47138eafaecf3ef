"""Per-kernel SASS instruction histogram of the built library (runs here, no
GPU): cuobjdump -sass, split by function, count opcodes (predicates and
modifiers stripped to the base mnemonic, e.g. DMMA.884 -> DMMA.884 kept as
the full opcode and DMMA as the family).

usage: python tools/sass_histogram.py [lib.so] [out.json]
"""
import collections
import json
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2203_02804_b200/libttpricer_b200.so"
out = sys.argv[2] if len(sys.argv) > 2 else "profiles/r02/sass_histogram.json"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
fn_re = re.compile(r"^\s*Function : (\S+)")
ins_re = re.compile(r"^\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)")
WATCH = ("DMMA", "DFMA", "DMUL", "DADD", "MUFU", "LDGSTS", "LDG", "STG", "LDS", "STS", "LDSM", "UTMALDG",
         "UTMASTG", "UBLKCP", "LDTM", "STTM", "UTCMMA", "UCGABAR", "ATOMS", "ATOMG", "RED", "SHFL", "BAR",
         "LDL", "STL")


def demangle(names):
    try:
        res = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True, check=True)
        return res.stdout.splitlines()
    except (OSError, subprocess.CalledProcessError):
        return names


kernels = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = fn_re.match(line)
    if m:
        cur = m.group(1)
        kernels.setdefault(cur, collections.Counter())
        continue
    m = ins_re.match(line)
    if m and cur:
        kernels[cur][m.group(2)] += 1
names = demangle(list(kernels))
result = {}
for (mangled, cnt), name in zip(kernels.items(), names):
    short = name.replace("(anonymous namespace)::", "").split("(")[0]
    fam = collections.Counter()
    for op, c in cnt.items():
        fam[op.split(".")[0].split("_")[0]] += c
    key = short if short not in result else f"{short} [{mangled[:60]}]"
    result[key] = {"total": sum(cnt.values()),
                   "families": {w: fam[w] for w in WATCH if fam[w]},
                   "top_opcodes": dict(cnt.most_common(25))}
with open(out, "w") as fh:
    json.dump({"library": lib, "tool": "cuobjdump -sass (CUDA 12.9) | tools/sass_histogram.py",
               "kernels": result}, fh, indent=1)
for k, v in result.items():
    if any(s in k for s in ("cluster_bond", "bond_kernel", "conv_site_dmma", "tt_inner_chunk", "fiber", "dense_partial")):
        print(f"{k[:70]:70s} {v['total']:7d} {v['families']}")
