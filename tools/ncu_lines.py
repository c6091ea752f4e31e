"""Attribute an ncu SASS source page (csv) to CUDA source lines via nvdisasm -g.
usage: python tools/ncu_lines.py <sass.csv> <nvdisasm -g output> <kernel mangled name> [top]"""
import csv, re, sys, collections
sass_csv, dis, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
addr2line = {}
cur = None; inside = False
for ln in open(dis):
    if '.section' in ln:
        inside = ('.text.' in ln) and (kern in ln)
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m and inside:
        cur = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+\S', ln)
    if m and inside and cur:
        addr2line[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]; data = rows[2:]
ai = hdr.index('Address'); ei = hdr.index('Instructions Executed'); si = hdr.index('Warp Stall Sampling (All Samples)')
src = hdr.index('Source')
ex = collections.Counter(); st = collections.Counter(); tot_e = tot_s = 0
base = min(int(r[ai], 16) for r in data if r and r[ai].startswith('0x'))
for r in data:
    try:
        a = int(r[ai], 16) - base; e = float(r[ei] or 0); s = float(r[si] or 0)
    except ValueError:
        continue
    key = addr2line.get(a, ('?', 0))
    ex[key] += e; st[key] += s; tot_e += e; tot_s += s
print(f"total instructions executed {tot_e:.3e}, stall samples {tot_s:.0f}; mapped lines {len(ex)}")
for key, v in sorted(st.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{key[0]}:{key[1]:<5d} stall {100*v/tot_s:5.1f}%  instr {100*ex[key]/tot_e:5.1f}%")
