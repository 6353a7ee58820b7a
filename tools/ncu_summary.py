"""Summarise an ncu report: headline metrics, stall mix, per-opcode stall attribution."""
import collections
import csv
import re
import subprocess
import sys

WANT = ['gpu__time_duration.sum', 'sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'lts__t_bytes.sum', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__inst_executed.sum', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__occupancy_limit_registers',
        'launch__occupancy_limit_shared_mem', 'sm__cycles_elapsed.avg.per_second']


def raw(rep):
    out = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[2]


def main(rep):
    h, v = raw(rep)
    for w in WANT:
        if w in h:
            print(f'{w:65s} {v[h.index(w)]}')
    out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[1]
    data = rows[2:]
    iSrc = h.index('Source')
    cols = [i for i, x in enumerate(h) if x.startswith('stall_') and 'Not Issued' not in x]
    agg = collections.defaultdict(collections.Counter)
    for r in data:
        m = re.match(r'\s*(@!?U?P\w+\s+)?([A-Z][A-Z0-9]*)', r[iSrc])
        op = m.group(2) if m else '?'
        for i in cols:
            try:
                agg[op][h[i]] += float(r[i] or 0)
            except ValueError:
                pass
    tot = collections.Counter()
    for op in agg:
        tot.update(agg[op])
    T = sum(tot.values()) or 1
    print('stalls:', {k[6:]: round(x / T * 100, 1) for k, x in tot.most_common(8)})
    byop = sorted(agg, key=lambda o: -sum(agg[o].values()))
    for op in byop[:8]:
        print(f'  {op:8s} {sum(agg[op].values()) / T * 100:5.1f}%',
              {k[6:]: round(x / T * 100, 1) for k, x in agg[op].most_common(4)})


if __name__ == '__main__':
    for rep in sys.argv[1:]:
        print('==', rep)
        main(rep)
