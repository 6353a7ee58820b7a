"""Per-opcode executed-instruction histogram of an ncu report (source page, SASS view):
warp-level instructions executed per opcode and their share -- the instruction mix of a kernel."""
import collections
import csv
import re
import subprocess
import sys


def opmix(rep, top=25):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    iSrc = h.index('Source')
    iEx = [i for i, x in enumerate(h) if x.startswith('Instructions Executed')][0]
    agg = collections.Counter()
    for r in rows[2:]:
        m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9]*(\.[A-Z0-9_]+)*)', r[iSrc])
        op = m.group(2).split('.')[0] if m else '?'
        try:
            agg[op] += float(r[iEx] or 0)
        except ValueError:
            pass
    T = sum(agg.values()) or 1
    print(f'total warp instructions executed: {T:.4g}')
    for op, n in agg.most_common(top):
        print(f'  {op:10s} {n:14.4g}  {n / T * 100:5.1f}%')
    return agg


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        print('==', rep)
        opmix(rep)
