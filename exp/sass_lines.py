"""Count SASS instructions (total, STL/LDL spills, DFMA...) per source line for one function
of an `nvdisasm --print-line-info` listing.  usage: sass_lines.py all.sass <function-substring> [top]"""
import collections
import re
import sys

path, fn = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
inside = False
cur = None
tot = collections.Counter()
stl = collections.Counter()
ldl = collections.Counter()
ops = collections.Counter()
for line in open(path):
    if line.startswith(".text."):
        inside = fn in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if not m:
        continue
    op = m.group(2)
    tot[cur] += 1
    ops[op.split(".")[0]] += 1
    if op.startswith("STL"):
        stl[cur] += 1
    if op.startswith("LDL"):
        ldl[cur] += 1
print("instructions", sum(tot.values()), "STL", sum(stl.values()), "LDL", sum(ldl.values()))
print("ops", ops.most_common(25))
byfile = collections.Counter()
for k, v in tot.items():
    byfile[k[0] if k else None] += v
print("by file", byfile.most_common())
print("STL by line", stl.most_common(top))
print("LDL by line", ldl.most_common(top))
