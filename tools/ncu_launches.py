"""Turn an `ncu --metrics ... --csv` launch list of bench.py into the files kept
under profiles/: a per-launch CSV and the per-layer DRAM traffic JSON that
bench.py reports as roofline.traffic.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size \\
        --clock-control none -s 6 -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1
    python tools/ncu_launches.py gpurun_out/launches.csv c2 round1 <unique_kv_bytes>
"""
import collections
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PAT_KERNELS = ("fwd_tc4_kernel", "fwd_stream_kernel", "merge_kernel")


def parse(path):
    rows = [r for r in csv.reader(open(path)) if r]
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    kernels = collections.OrderedDict()
    for r in rows[start + 1:]:
        d = dict(zip(hdr, r))
        k = kernels.setdefault(d["ID"], {"kernel": d["Kernel Name"], "grid": d.get("Grid Size", ""),
                                          "block": d.get("Block Size", "")})
        val = float(d["Metric Value"].replace(",", "")) if d["Metric Value"] else 0.0
        unit = d.get("Metric Unit", "")
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e3, "msecond": 1e6,
                 "nsecond": 1.0}.get(unit, 1.0)
        k[d["Metric Name"]] = val * scale
    return list(kernels.values())


def main(path, config, rnd, unique_bytes, cmd="bench.py"):
    ks = parse(path)
    out_csv = os.path.join(REPO, "profiles", f"{rnd}_launches_{config}.csv")
    with open(out_csv, "w") as fh:
        fh.write(f"# {rnd} -- ncu launch list, {cmd} {config} (ncu --metrics gpu__time_duration.sum,"
                 "dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none)\n")
        fh.write("# per-launch times are cold-cache and serialised under ncu: compare SHARES, not absolutes\n")
        fh.write("id,kernel,grid,block,time_ns,dram_read_bytes,dram_write_bytes\n")
        for i, k in enumerate(ks):
            name = k["kernel"].replace(",", ";")[:60]
            fh.write(f"{i},{name},{k['grid']},{k['block']},{k.get('gpu__time_duration.sum', 0):.0f},"
                     f"{k.get('dram__bytes_read.sum', 0):.0f},{k.get('dram__bytes_write.sum', 0):.0f}\n")
    pat = [k for k in ks if any(p in k["kernel"] for p in PAT_KERNELS)]
    # one layer = one launch of each distinct PAT kernel; average over the layers seen
    per = collections.defaultdict(list)
    for k in pat:
        name = next(p for p in PAT_KERNELS if p in k["kernel"])
        per[name].append(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0))
    per_kernel = {n: sum(v) / len(v) for n, v in per.items()}
    times = collections.defaultdict(list)
    for k in pat:
        name = next(p for p in PAT_KERNELS if p in k["kernel"])
        times[name].append(k.get("gpu__time_duration.sum", 0))
    res = {
        "workload": config,
        "source": os.path.relpath(out_csv, REPO) + " (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum, "
                                                   f"{cmd} layers)",
        "layer_dram_bytes": sum(per_kernel.values()),
        "algorithmic_unique_kv_bytes": unique_bytes,
        "per_kernel_dram_bytes": per_kernel,
        "per_kernel_ncu_time_ns": {n: sum(v) / len(v) for n, v in times.items()},
    }
    out_json = os.path.join(REPO, "profiles", f"{rnd}_traffic_{config}.json")
    json.dump(res, open(out_json, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4]), *sys.argv[5:6])
