"""Attribute ncu per-SASS-instruction stall samples to functions and source
lines (needs `ncu --page source --csv --print-source sass` output and
`nvdisasm -g` of the cubin). Usage:
  python profiles/sass_hotspots.py <ncu_source_sass.csv> <nvdisasm.sass> <mangled kernel>
"""
import collections
import csv
import re
import sys


def load_ncu(path):
    r = list(csv.reader(open(path)))
    for i, row in enumerate(r):
        if 'Address' in row and 'Source' in row:
            hdr, rows = row, r[i + 1:]
            break
    iss, iex = hdr.index('Warp Stall Sampling (All Samples)'), hdr.index('Instructions Executed')
    out = []
    for x in rows:
        try:
            out.append((float(x[iss] or 0), float(x[iex] or 0)))
        except (ValueError, IndexError):
            continue
    return out


def load_sass(path, kernel):
    out, cur_func, cur_line, inside = [], kernel, None, False
    for line in open(path):
        if line.startswith('\t.section') or line.startswith('.section'):
            inside = ('.text.' + kernel) in line
            continue
        if not inside:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', line)
        if m:
            cur_line = m.group(1).split('/')[-1] + ':' + m.group(2)
            continue
        m = re.match(r'^\s*\.?\$?([A-Za-z_$][\w$@]*):', line)
        if m and 'ZN' in m.group(1):
            name = m.group(1).split('$')[-1]
            cur_func = name
            continue
        if re.search(r'/\*[0-9a-f]{4,}\*/\s+[^\s]', line) and not line.strip().startswith('.'):
            out.append((cur_func, cur_line))
    return out


def main():
    ncu, sass, kernel = sys.argv[1:4]
    samples = load_ncu(ncu)
    ins = load_sass(sass, kernel)
    n = min(len(samples), len(ins))
    print(f"ncu rows {len(samples)}, sass instructions {len(ins)}")
    tot = sum(s for s, _ in samples) or 1
    byf, byl, exf = collections.Counter(), collections.Counter(), collections.Counter()
    for (s, e), (f, l) in zip(samples[:n], ins[:n]):
        byf[f] += s
        byl[l] += s
        exf[f] += e
    print("by function (stall-sample share, executed warp instructions):")
    for f, s in byf.most_common(20):
        print(f"  {100 * s / tot:5.1f}%  {exf[f] / 1e6:9.1f}M  {f}")
    print("by source line:")
    for l, s in byl.most_common(30):
        print(f"  {100 * s / tot:5.1f}%  {l}")


if __name__ == "__main__":
    main()
