"""Summarise ncu outputs into profiles/ (committed evidence).

    python tools/ncu_summary.py launches <launches.csv> <out.txt>
    python tools/ncu_summary.py full <report.ncu-rep> <out.txt>
"""
import collections
import csv
import subprocess
import sys


def launches(path, out):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start:]:
        name = r[ik].split("(")[0].replace("void ", "")
        v = float(r[iv].replace(",", ""))
        u = r[iu]
        v = v / 1e3 if u in ("nsecond", "ns") else (v * 1e3 if u in ("msecond", "ms") else v)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(x[1] for x in agg.values())
    with open(out, "w") as fh:
        fh.write(f"# ncu launch list (gpu__time_duration.sum, cold-cache serialised): {path}\n")
        fh.write(f"{'kernel':60s} {'launches':>8s} {'total_us':>12s} {'avg_us':>10s} {'share':>7s}\n")
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"{k[:60]:60s} {c:8d} {v:12.1f} {v / c:10.1f} {100 * v / tot:6.1f}%\n")
        fh.write(f"{'TOTAL':60s} {sum(x[0] for x in agg.values()):8d} {tot:12.1f}\n")


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "smsp__inst_executed_op_shared_atom.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "lts__t_sectors_op_red.sum", "l1tex__t_bytes_pipe_lsu_mem_global_op_ld.sum"]


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full summary: {path}\n")
        for r in rows[2:]:
            name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
            fh.write(f"\n## {name[:120]}\n")
            for m in WANT:
                if m in hdr:
                    fh.write(f"{m:70s} {r[hdr.index(m)]}\n")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"):
                try:
                    stalls.append((h, float(rows[2][i].replace(",", ""))))
                except (ValueError, IndexError):
                    pass
        stalls.sort(key=lambda x: -x[1])
        fh.write("\n# top stall reasons (first kernel, pc samples)\n")
        for h, v in stalls[:8]:
            fh.write(f"{h:70s} {v:.0f}\n")


def traffic(path, out):
    """dram bytes (read + write) per launch of the captured kernels -> JSON for bench.py's roofline"""
    import json
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    vals = []
    for r in rows[2:]:
        b = 0.0
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            v = float(r[hdr.index(m)].replace(",", ""))
            u = units[hdr.index(m)]
            b += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        vals.append(b)
    json.dump({"source": path, "launches": len(vals), "dram_bytes_per_launch": sum(vals) / max(1, len(vals)),
               "per_launch": vals}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full, "traffic": traffic}[sys.argv[1]](sys.argv[2], sys.argv[3])
