"""Summarise an ncu report (details page + key raw metrics) as text.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [--raw] [--source]
"""
import csv
import io
import subprocess
import sys


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def details(rep):
    out = ncu("-i", rep, "--page", "details", "--csv")
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    si, mi, ui, vi = (hdr.index(x) for x in ("Section Name", "Metric Name", "Metric Unit", "Metric Value"))
    ki = hdr.index("Kernel Name")
    last = None
    lines = []
    for r in rows[1:]:
        if len(r) <= vi or not r[mi]:
            continue
        if r[ki] != last:
            lines.append(f"== {r[ki][:120]}")
            last = r[ki]
        lines.append(f"{r[si][:28]:28s} | {r[mi][:60]:60s} | {r[vi]:>16s} {r[ui]}")
    return "\n".join(lines)


RAW_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
            "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def raw(rep):
    out = ncu("-i", rep, "--page", "raw", "--csv")
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    lines = []
    for r in rows[2:]:
        for k in RAW_KEYS:
            if k in hdr:
                i = hdr.index(k)
                lines.append(f"{k:75s} {r[i]:>18s} {units[i]}")
    return "\n".join(lines)


def source(rep, top=25):
    out = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    rows = list(csv.reader(io.StringIO(out)))
    rows = [r for r in rows if len(r) > 3]
    if not rows:
        return ""
    hdr = rows[0]
    try:
        si = hdr.index("Source")
        wi = [i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All")][0]
    except (ValueError, IndexError):
        return "source page unavailable"
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[wi] or 0), r[si]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1
    data.sort(reverse=True)
    return "\n".join(f"{100 * w / tot:6.2f}%  {s[:110]}" for w, s in data[:top])


def source_ordered(rep):
    """Every SASS line with its stall-sample share, in program order."""
    out = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    rows = [r for r in csv.reader(io.StringIO(out)) if len(r) > 3]
    hdr = rows[0]
    si = hdr.index("Source")
    wi = [i for i, h in enumerate(hdr) if h.startswith("Warp Stall Sampling (All")][0]
    tot = sum(float(r[wi] or 0) for r in rows[1:]) or 1
    return "\n".join(f"{100 * float(r[wi] or 0) / tot:6.2f}%  {r[si][:110]}" for r in rows[1:])


if __name__ == "__main__":
    rep = sys.argv[1]
    print(details(rep))
    if "--raw" in sys.argv:
        print(raw(rep))
    if "--source" in sys.argv:
        print(source(rep))
    if "--sass" in sys.argv:
        print(source_ordered(rep))
