"""Per-kernel SASS instruction summary of libpmg_cuda.so (cuobjdump -sass):
registers, code size and the counts of the instructions that identify the
hardware paths -- DMMA (FP64 tensor cores), UBLKCP (cp.async.bulk / TMA),
LDGSTS (cp.async), SYNCS (mbarrier), LDS/STS, DFMA, BAR.

  python scripts/sass_summary.py [lib] > profiles/sass_summary_rNN.txt
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1804_02539_b200/lib/libpmg_cuda.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
regs = {}
cur = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        cur = m.group(1)
    m = re.search(r"REG:(\d+) .*SHARED:(\d+)", line)
    if m and cur:
        regs[cur] = (int(m.group(1)), int(m.group(2)))
demangle = subprocess.run(["c++filt"], input="\n".join(regs), capture_output=True, text=True).stdout.splitlines()
names = dict(zip(regs, demangle))
KEYS = ["DMMA", "UBLKCP", "LDGSTS", "SYNCS", "LDS", "STS", "DFMA", "BAR", "LDG", "STG", "ATOM"]
counts = collections.defaultdict(collections.Counter)
total = collections.Counter()
cur = None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\d+\s+)?([A-Z0-9_]+)", line)
    if m and cur:
        op = m.group(1)
        total[cur] += 1
        for k in KEYS:
            if op == k or op.startswith(k + "."):
                counts[cur][k] += 1
        if op.startswith("ATOM") or op.startswith("RED"):
            counts[cur]["ATOM"] += 1
print(f"# SASS summary of {lib} (sm_100a; cuobjdump -sass, static instruction counts per kernel)")
print(f"{'kernel':78s} {'regs':>4s} {'instr':>6s} " + " ".join(f"{k:>6s}" for k in KEYS))
short = lambda n: re.sub(r"\(.*", "", re.sub(r"pmgcu::\(anonymous namespace\)::|void ", "", n))
for f in sorted(total, key=lambda f: short(names.get(f, f))):
    print(f"{short(names.get(f, f))[:78]:78s} {regs.get(f, (0, 0))[0]:4d} {total[f]:6d} " +
          " ".join(f"{counts[f][k]:6d}" for k in KEYS))
