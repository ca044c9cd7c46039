"""Map an ncu SASS source page (--page source --csv --print-source sass) to CUDA
source lines using nvdisasm -g of the same cubin; print the top stall lines.
usage: python scripts/ncu_lines.py SOURCE_SASS_CSV NVDISASM_G_OUTPUT FUNC_SUBSTR"""
import collections, csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
base = int(data[0]["Address"], 16)
amap, line, infn = {}, None, False
for l in open(sys.argv[2]):
    m = re.match(r"^(\S+):\s*$", l)
    if m and not m.group(1).startswith(".L_x"):
        infn = sys.argv[3] in m.group(1)
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
    m = re.match(r"\s*/\*([0-9a-f]+)\*/", l)
    if m and infn:
        amap[int(m.group(1), 16)] = line
bl, tot = collections.Counter(), 0
for d in data:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    tot += s
    bl[amap.get(int(d["Address"], 16) - base)] += s
print("samples", tot)
for k, v in bl.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 30):
    print(f"{v:6.0f} {100 * v / tot:5.1f}% {k}")
