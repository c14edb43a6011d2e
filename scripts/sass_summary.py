"""Static SASS instruction counts per kernel of libswarm_b200.so (tcgen05 / TMA evidence):
   python scripts/sass_summary.py > profiles/<round>_sass_summary.md"""
import collections
import re
import subprocess
import sys

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2301_11913_b200/libswarm_b200.so"
KEYS = ["UTCHMMA", "UTCQMMA", "UTMALDG", "UTMASTG", "UTMAREDG", "UTMAPF", "LDTM", "UTCBAR", "MUFU.TANH", "MUFU.EX2",
        "FFMA", "REDG", "SYNCS"]
sass = subprocess.run(f"cuobjdump -sass {LIB} | c++filt", shell=True, capture_output=True, text=True).stdout
counts, name = collections.OrderedDict(), None
for line in sass.splitlines():
    m = re.match(r"\s*Function : (.*)", line)
    if m:
        name = m.group(1).strip()
        counts[name] = collections.Counter()
        continue
    if name is None:
        continue
    ins = re.search(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
    if not ins:
        continue
    op = ins.group(1)
    for k in KEYS:
        if op == k or op.startswith(k + "."):
            counts[name][k] += 1
rows = [(n, c) for n, c in counts.items() if any(c[k] for k in ("UTCHMMA", "UTMALDG", "UTMASTG", "UTMAREDG", "LDTM"))]
print("# SASS instruction summary of libswarm_b200.so (sm_100a)\n")
print(f"`python scripts/sass_summary.py` = `cuobjdump -sass {LIB} | c++filt`, static counts per kernel:")
print("UTCHMMA = tcgen05.mma (bf16), UTMALDG / UTMASTG / UTMAREDG / UTMAPF = TMA load / store / reduce-add / L2")
print("prefetch, LDTM = tcgen05.ld (TMEM -> registers), UTCBAR = tcgen05.commit, SYNCS = mbarrier ops, REDG =")
print("global reductions.  Kernels with no tcgen05 / TMA instruction are omitted.\n")
print("| kernel | " + " | ".join(KEYS) + " |")
print("|---|" + "---:|" * len(KEYS))
for n, c in rows:
    short = re.sub(r"\(.*", "", n).replace("void ", "").replace("swarm::", "")
    print(f"| `{short}` | " + " | ".join(str(c[k]) for k in KEYS) + " |")
