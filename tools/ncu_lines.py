"""Attribute ncu's per-SASS-instruction execution counts to CUDA source lines (nvdisasm -g line table).
usage: ncu_lines.py <sass.csv from ncu --page source --print-source=sass> <nvdisasm -g output> <mangled kernel> <src>"""
import csv, re, sys
sass_csv, lines_txt, kern, srcfile = sys.argv[1:5]
txt = open(lines_txt).read().split('\n')
start = None
for i, l in enumerate(txt):
    if '.text.' + kern in l and ('.section' in l or l.strip().endswith(':')):
        start = i
        break
off2line, line = {}, None
for l in txt[start + 1:]:
    if '.section' in l and '.text.' in l and kern not in l:
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split('/')[-1], int(m.group(2)))
        continue
    m = re.match(r'\s*/\*([0-9a-f]+)\*/', l)
    if m and line:
        off2line[int(m.group(1), 16)] = line
rows = list(csv.reader(open(sass_csv)))
hdr, data = rows[1], rows[2:]
ie, ad = hdr.index('Instructions Executed'), hdr.index('Address')
th = hdr.index('Thread Instructions Executed') if 'Thread Instructions Executed' in hdr else None
base, agg, tot = None, {}, 0
for r in data:
    try:
        n = int(r[ie] or 0); a = int(r[ad], 16)
    except ValueError:
        continue
    if base is None:
        base = a
    ln = off2line.get(a - base, ('?', 0))
    agg[ln] = agg.get(ln, 0) + n
    tot += n
import os
srcdir = os.path.dirname(os.path.abspath(srcfile))
_cache = {}
def src_line(f, l):
    if f not in _cache:
        try:
            _cache[f] = open(os.path.join(srcdir, f)).read().split('\n')
        except OSError:
            _cache[f] = []
    s = _cache[f]
    return s[l - 1].strip()[:90] if 0 < l <= len(s) else ''
print("total warp-level instructions", tot)
for (f, l), n in sorted(agg.items(), key=lambda x: -x[1])[:int(sys.argv[5]) if len(sys.argv) > 5 else 40]:
    s = src_line(f, l)
    print("%5.2f%% %-22s %4d  %s" % (100.0 * n / tot, f, l, s))
