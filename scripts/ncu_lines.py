"""Per-source-line executed-instruction counts of one kernel in an ncu report (SASS page
joined with nvdisasm line info). usage: ncu_lines.py REPORT CUBIN_OBJ MANGLED [per_unit]"""
import csv, collections, re, subprocess, sys, os, tempfile
rep, obj, fn = sys.argv[1:4]
unit = float(sys.argv[4]) if len(sys.argv) > 4 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith(f".text.{fn}:"))
a2l, cur = {}, None
for l in txt[start + 1:]:
    if l.startswith(".text."):
        break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and cur:
        a2l[int(m.group(1), 16)] = cur
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]
ie, smp = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
sidx = hdr.index("Source")
base = int(rows[2][0], 16)
cnt, ss, ops = collections.Counter(), collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        a, n, s = int(r[0], 16) - base, int(r[ie]), int(r[smp])
    except (ValueError, IndexError):
        continue
    k = a2l.get(a, ("?", 0))
    cnt[k] += n
    ss[k] += s
    op = re.sub(r"^@!?U?P\w+\s+", "", r[sidx].strip()).split(" ")[0].split(".")[0]
    ops[op] += n
tot, tots = sum(cnt.values()), sum(ss.values())
print(f"total warp instructions {tot} ({tot / unit:.1f} per unit)")
for op, n in ops.most_common(16):
    print(f"  {op:8s} {n / unit:8.1f}")
for k, n in cnt.most_common(30):
    print(f"{n / unit:8.1f} {100 * ss[k] / tots:5.1f}% {k}")
