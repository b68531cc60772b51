#!/usr/bin/env python
"""Summarise ncu outputs into profiles/*.md (run here, no GPU needed).

  python tools/ncu_summary.py launches <launches.csv>        # per-kernel share of device time
  python tools/ncu_summary.py full <report.ncu-rep>          # key counters of one captured launch
  python tools/ncu_summary.py source <report.ncu-rep> [N]    # top-N source lines by stall samples
  python tools/ncu_summary.py mix <report.ncu-rep>           # SASS opcode mix: executed, stall samples, smem
"""
import collections
import csv
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def short(name):
    n = name.split("(")[0]
    return n.split("::")[-1].replace("void ", "").strip()


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.Counter(), collections.Counter()
    for r in rows[1:]:
        v = float(r[mi].replace(",", "")) * UNIT.get(r[ui], 1.0)
        tot[short(r[ki])] += v
        cnt[short(r[ki])] += 1
    T = sum(tot.values())
    print("| kernel | launches | total us | avg us | share of device time |")
    print("|---|---|---|---|---|")
    for n, v in tot.most_common():
        print("| %s | %d | %.1f | %.2f | %.3f |" % (n, cnt[n], v, v / cnt[n], v / T))


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__cycles_elapsed.avg.per_second"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    print("kernel: %s" % short(v[h.index("Kernel Name")]))
    print()
    print("| counter | value | unit |")
    print("|---|---|---|")
    for k in KEYS:
        if k in h:
            i = h.index(k)
            print("| %s | %s | %s |" % (k, v[i], units[i]))
    st = []
    for i, n in enumerate(h):
        if n.startswith("smsp__average_warps_issue_stalled") and n.endswith("per_issue_active.ratio"):
            try:
                st.append((float(v[i]), n.split("stalled_")[1].split("_per")[0]))
            except ValueError:
                pass
    print()
    print("warp stall reasons (cycles per issued instruction): " +
          ", ".join("%s %.2f" % (n, x) for x, n in sorted(st, reverse=True)[:8]))


def source(path, top=15):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if len(r) > 4 and r[0] == "Line No"][0]
    h = rows[hi]
    S = h.index("Warp Stall Sampling (All Samples)")
    names = [n for n in h if n.startswith("stall_") and "Not Issued" not in n]
    cols = {n: i for i, n in enumerate(h)}
    by, byst, text = collections.Counter(), collections.defaultdict(collections.Counter), {}
    cur = None
    for r in rows[hi + 1:]:
        if len(r) <= S:
            continue
        if r[0]:
            cur = r[0]
            text[cur] = r[1]
        try:
            by[cur] += int(r[S])
        except ValueError:
            continue
        for n in names:
            try:
                byst[cur][n] += int(r[cols[n]])
            except ValueError:
                pass
    T = sum(by.values())
    print("| share | line | source | top stalls |")
    print("|---|---|---|---|")
    for ln, x in by.most_common(top):
        st = ", ".join("%s %d" % (k[6:], c) for k, c in byst[ln].most_common(3))
        print("| %.1f%% | %s | `%s` | %s |" % (100.0 * x / T, ln, text.get(ln, "").strip()[:80].replace("|", "\\|"), st))


def mix(path, top=20):
    out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = [i for i, r in enumerate(rows) if len(r) > 4 and r[0] == "Address"][0]
    h = rows[hi]
    ix = {n: i for i, n in enumerate(h)}
    ex, sm, wf = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) < len(h):
            continue
        src = r[ix["Source"]].split()
        if not src:
            continue
        op = (src[1] if src[0].startswith("@") and len(src) > 1 else src[0]).split(".")[0]
        ex[op] += int(r[ix["Instructions Executed"]] or 0)
        sm[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        wf[op] += int(r[ix["L1 Wavefronts Shared"]] or 0)
    TE, TS = sum(ex.values()), sum(sm.values())
    print("| opcode | warp instructions executed | share | stall samples | share | shared wavefronts |")
    print("|---|---|---|---|---|---|")
    for op, c in ex.most_common(top):
        print("| %s | %d | %.1f%% | %d | %.1f%% | %d |" % (op, c, 100.0 * c / TE, sm[op], 100.0 * sm[op] / max(TS, 1), wf[op]))


if __name__ == "__main__":
    {"launches": launches, "full": full, "source": source, "mix": mix}[sys.argv[1]](*sys.argv[2:3])
