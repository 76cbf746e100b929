"""Executed-instruction mix of one kernel from an ncu report's SASS source
page: warp instructions and stall samples per opcode class, per source file
region, and the top source lines.

usage: ncu_sass_mix.py report.ncu-rep [regions.json]
regions: {"name": ["file.cuh", first_line, last_line], ...}
"""
import collections
import csv
import json
import re
import subprocess
import sys

rep = sys.argv[1]
regions = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else {}
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))

CLASSES = [
    ("fp64", re.compile(r"^(DFMA|DADD|DMUL|DSETP|DMNMX|DSET)")),
    ("f2f/i2f", re.compile(r"^(F2F|I2F|F2I|FRND)")),
    ("mufu", re.compile(r"^MUFU")),
    ("fp32", re.compile(r"^(FFMA|FADD|FMUL|FSETP|FMNMX|FSEL|FSET|FCHK)")),
    ("lds", re.compile(r"^(LDS|LDSM)")),
    ("sts", re.compile(r"^STS")),
    ("local", re.compile(r"^(LDL|STL)")),
    ("global", re.compile(r"^(LDG|STG|ATOMG|RED|ATOM|LD\b|ST\b)")),
    ("uniform", re.compile(r"^(U[A-Z0-9]+|LDC|LDCU|S2UR|R2UR)")),
    ("branch", re.compile(r"^(BRA|BSSY|BSYNC|EXIT|CALL|RET|WARPSYNC|BREAK|BPT)")),
    ("shfl/vote", re.compile(r"^(SHFL|VOTE|MATCH)")),
    ("sync", re.compile(r"^(SYNCS|BAR|MEMBAR|FENCE|NANOSLEEP|CCTL)")),
]


def opclass(op):
    for name, rx in CLASSES:
        if rx.match(op):
            return name
    return "int/other"


hdr = None
fname = None
cur_line = None
by_cls = collections.Counter()
st_cls = collections.Counter()
by_reg = collections.defaultdict(collections.Counter)
by_line = collections.Counter()
st_line = collections.Counter()
src = {}
ops = collections.Counter()
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur_line = (fname, int(r[0]))
        src[cur_line] = r[1]
        continue
    if r[2] in ("...", "-") or not r[2].startswith("0x"):
        continue
    d = dict(zip(hdr[:4], r[:4]))
    sass = r[3].strip()
    op = sass.split()[0]
    if op.startswith("@"):
        op = sass.split()[1]
    try:
        n = int(r[7])
        stall = float(r[4])
    except ValueError:
        continue
    base = op.split(".")[0]
    c = opclass(base)
    by_cls[c] += n
    st_cls[c] += stall
    ops[base] += n
    by_line[cur_line] += n
    st_line[cur_line] += stall
    reg = "other"
    for name, (f, a, b) in regions.items():
        if cur_line and cur_line[0] == f and a <= cur_line[1] <= b:
            reg = name
            break
    by_reg[reg][c] += n
    by_reg[reg]["_stall"] += stall

tot = sum(by_cls.values())
tst = sum(st_cls.values())
print(f"warp instructions {tot:,}  stall samples {tst:,.0f}")
print("\n-- opcode classes (share of executed warp instructions / of stall samples)")
for c, n in by_cls.most_common():
    print(f"  {c:10s} {n / tot * 100:5.1f}%  {st_cls[c] / tst * 100:5.1f}%")
print("\n-- top opcodes")
for o, n in ops.most_common(25):
    print(f"  {o:10s} {n / tot * 100:5.1f}%")
if regions:
    print("\n-- regions: instr share, stall share, fp64 share of region")
    for name, cnt in sorted(by_reg.items(), key=lambda kv: -sum(v for k, v in kv[1].items() if k != "_stall")):
        n = sum(v for k, v in cnt.items() if k != "_stall")
        print(f"  {name:22s} {n / tot * 100:5.1f}%  {cnt['_stall'] / tst * 100:5.1f}%  fp64 {cnt['fp64'] / max(n, 1) * 100:4.0f}%"
              f"  lds {cnt['lds'] / max(n, 1) * 100:3.0f}%  local {cnt['local']:,}")
print("\n-- top source lines by executed instructions")
for k, n in by_line.most_common(30):
    print(f"  {n / tot * 100:5.1f}% st {st_line[k] / tst * 100:4.1f}%  {k[0][:12]}:{k[1]:<4d} {src.get(k, '')[:80]}")
