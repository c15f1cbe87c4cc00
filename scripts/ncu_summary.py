"""Summarise an ncu --set full report of the decode kernel (metrics + stall mix).
usage: python scripts/ncu_summary.py report.ncu-rep [--source]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_elapsed",
        "sm__cycles_elapsed.avg", "sm__cycles_active.avg", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
for r in rows[2:]:
    print("-" * 60)
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"{w:62s} {r[i][:70]:>20s} {units[i]}")
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), r[i]) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
    st = [(n, float(v.replace(",", ""))) for n, v in st if v]
    tot = sum(v for _, v in st) or 1
    print("stalls:", ", ".join(f"{n} {100*v/tot:.0f}%" for n, v in sorted(st, key=lambda x: -x[1])[:8]))
    break
if "--source" in sys.argv:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(src)))
    h = rr[1]
    ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
    seen, data = set(), []
    for r in rr[2:]:
        if len(r) < len(h) or r[ia] in seen:
            continue
        seen.add(r[ia])
        try:
            data.append((int(r[iall] or 0), r[ia], r[isrc].strip()))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    for s, a, t in sorted(data, reverse=True)[:20]:
        print(f"{100*s/tot:5.1f}% {a} {t}")
