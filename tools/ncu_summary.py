"""Summarise an ncu report (--set full) into the text kept under profiles/."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_op_hmma.avg.pct_of_peak_sustained_active",
        "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def stalls(rep, top=8):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    tot = sum(float(r[ist] or 0) for r in data) or 1
    best = sorted(range(len(data)), key=lambda i: -float(data[i][ist] or 0))[:top]
    return [f"{float(data[i][ist]) / tot * 100:5.1f}%  {data[i][isrc].strip()[:70]}   (after: {data[i-1][isrc].strip()[:40]})"
            for i in best]


def main(rep, title):
    v, units = raw(rep)
    print(f"# {title}\n# source: {rep}\n")
    print(f"kernel: {v.get('Kernel Name', '?')[:120]}")
    for k in KEYS:
        if k in v:
            print(f"{k:75s} {v[k]:>16s} {units.get(k, '')}")
    print("\nTop stall sites (warp-stall sampling, all samples):")
    for s in stalls(rep):
        print("  " + s)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
