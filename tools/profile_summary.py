"""Write a round's profile summary (markdown) from the bench JSON, the ncu launch list and one
ncu --set full capture of the transport kernel:
  python tools/profile_summary.py TAG OUT.md   (reads gpurun_out/TAG_{bench.json,launches.csv,transport.ncu-rep})
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h, start = r, i
            break
    iK, iV, iN = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    c = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) > iV and r[iN] == "gpu__time_duration.sum":
            name = r[iK].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]
            c[name].append(float(r[iV].replace(",", "")))
    return c


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return dict(zip(r[0], r[2]))


def main(tag, out_md):
    b = json.load(open(f"gpurun_out/{tag}_bench.json"))
    L = launches(f"gpurun_out/{tag}_launches.csv")
    m = raw(f"gpurun_out/{tag}_transport.ncu-rep")
    tot = sum(sum(v) for v in L.values())
    lines = [f"# {tag} -- C5 (40^3 particles x 25^3 velocity nodes, ALE, particle management on), one B200", "",
             f"Bench (`python bench.py --steps 10 --warmup 3`, `profiles/{tag}_bench.json`): "
             f"**{b['ms_per_step']:.1f} ms/step, {b['value']:.3e} particle-velocity updates/s**; SM clock median "
             f"{b['clocks']['sm_mhz']:.0f} MHz (max {b['clocks']['sm_max_mhz']:.0f}), reasons {b['clocks']['reasons']}; "
             f"e2e through the C ABI with the 8 GB state copied from pinned host memory every step: "
             f"{b['e2e']['value']:.3e} updates/s.  CPU oracle on the same box ({b['cpu_baseline']['cores']} threads, "
             f"bounded sample): {b['cpu_baseline']['value']:.3e} updates/s.", "",
             f"Phases (CUDA events): " + ", ".join(f"{k} {v:.2f} ms" for k, v in b["phases_ms"].items()), "",
             "Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, bench with --steps 2 "
             f"--warmup 1, `profiles/{tag}_launches.csv`; cold-cache, serialised):", "",
             "| kernel | launches | ms/launch | share |", "|---|---|---|---|"]
    for k, v in sorted(L.items(), key=lambda kv: -sum(kv[1])):
        if sum(v) / tot < 0.001:
            continue
        lines.append(f"| {k} | {len(v)} | {sum(v) / len(v) / 1e6:.3f} | {sum(v) / tot * 100:.1f} % |")
    dr = float(m["dram__bytes_read.sum"]) * (1e9 if float(m["dram__bytes_read.sum"]) < 1e6 else 1)
    dw = float(m["dram__bytes_write.sum"]) * (1e9 if float(m["dram__bytes_write.sum"]) < 1e6 else 1)
    lines += ["", f"`ncu --set full` of k_transport (one launch, `gpurun_out/{tag}_transport.ncu-rep`):",
              f"- duration {float(m['gpu__time_duration.sum']):.2f} ms; fp64 pipe "
              f"{float(m['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']):.1f} %, issue slots "
              f"{float(m['smsp__issue_active.avg.pct_of_peak_sustained_active']):.1f} %, "
              f"{float(m['launch__registers_per_thread']):.0f} registers, warps active "
              f"{float(m['sm__warps_active.avg.pct_of_peak_sustained_active']):.1f} %;",
              f"- DRAM read {dr / 1e9:.1f} GB + write {dw / 1e9:.1f} GB per launch (`roofline.traffic`); "
              f"L2 throughput {float(m['lts__throughput.avg.pct_of_peak_sustained_elapsed']):.1f} % of ncu's peak;",
              f"- roofline line (bench): {b['roofline']['achieved']:.2f} of {b['roofline']['peak']:.2f} "
              f"{b['roofline']['unit']} -> frac {b['roofline']['frac']:.3f} ({b['roofline']['per_unit']})."]
    open(out_md, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
