"""Warp-stall samples and executed instructions per CUDA source line for one kernel.

    python tools/line_profile.py report.ncu-rep|source.csv build/obj/<unit>.o <kernel-regex> <mangled-substring> [n]

(a .csv argument is an `ncu -i rep --page source --csv -k <kernel>` export)

Maps the ncu SASS page (absolute addresses) onto `nvdisasm -g` line info of the
same object's cubin (function-relative offsets)."""
import collections, csv, glob, io, os, re, subprocess, sys, tempfile

rep, obj, kre, mangled = sys.argv[1:5]
n = int(sys.argv[5]) if len(sys.argv) > 5 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
start = [m.start() for m in re.finditer(r"\.text\.\S*" + re.escape(mangled), txt)][0]
body = txt[start:]
nxt = body.find("//---------------------", 10)
body = body[:nxt] if nxt > 0 else body
line, off2line = None, {}
for l in body.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", l)
    if m and line:
        off2line[int(m.group(1), 16)] = line
if rep.endswith(".csv"):
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", "regex:" + kre], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:  # the first launch's section only
    if len(r) == len(hdr) and r[idx["Address"]] == "Address":
        break
    if len(r) == len(hdr):
        data.append(r)
base = min(int(r[idx["Address"]], 16) for r in data)
S = "Warp Stall Sampling (All Samples)"
tot = sum(int(r[idx[S]] or 0) for r in data)
agg, ins = collections.Counter(), collections.Counter()
for r in data:
    ln = off2line.get(int(r[idx["Address"]], 16) - base, ("?", 0))
    agg[ln] += int(r[idx[S]] or 0)
    ins[ln] += int(r[idx["Instructions Executed"]] or 0)
print(f"{tot} samples, {sum(ins.values())/1e6:.1f}M warp instructions")
for (f, k), s in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{100*s/tot:5.1f}% {ins[(f, k)]/1e6:7.2f}M {f}:{k}")
