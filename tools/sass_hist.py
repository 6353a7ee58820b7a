"""Static SASS opcode histogram of one kernel of the built library (cuobjdump -sass): the instruction
mix the compiler emitted -- e.g. the fp64 (DFMA/DADD), integer-pipe (VIMNMX), shared-memory (LDS),
TMA (UTMALDG/UBLKCP) and mbarrier (SYNCS) instructions of k_transport<3, 25>.

    python tools/sass_hist.py [substring of the mangled kernel name] [library or object]
"""
import collections
import re
import subprocess
import sys


def kernels(path):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    cur, body = None, collections.OrderedDict()
    for ln in out.splitlines():
        m = re.search(r"Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            body[cur] = []
            continue
        if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
            body[cur].append(ln)
    return body


def hist(lines):
    h = collections.Counter()
    for ln in lines:
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", ln)
        if m:
            h[m.group(2)] += 1
    return h


def main():
    pat = sys.argv[1] if len(sys.argv) > 1 else "k_transportILi3ELi25ELi4ELi2ELb0E"
    path = sys.argv[2] if len(sys.argv) > 2 else "paper_2408_02350_b200/libbgk_b200.so"
    for name, lines in kernels(path).items():
        if pat in name:
            h = hist(lines)
            tot = sum(h.values())
            print(f"{name}: {tot} SASS instructions")
            for op, n in h.most_common(40):
                print(f"  {op:12s} {n:6d}  {100 * n / tot:5.1f}%")


if __name__ == "__main__":
    main()
