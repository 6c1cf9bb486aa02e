"""Summarise an ncu per-launch metrics CSV (gpu__time_duration, dram bytes) into
profiles/ncu_traffic.json (read by bench.py for roofline.traffic).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none -k regex:"gemm|sample_qrcp|panel" --csv --log-file X.csv \
        python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline
    python tools/ncu_traffic.py X.csv profiles/ncu_traffic.json
"""
import collections
import csv
import json
import sys

M = N = 32768
B = 128


def algorithmic_bytes():
    """C5 streaming bytes per kernel class: every block's first sweep reads its
    trailing matrix once (Y^T C); the second sweep runs once per block PAIR
    (driver.cu trailing_second, K = 2b) and reads + writes the second block's
    trailing matrix; the sketch reads A once."""
    c = sum((M - B * j) * (N - B * (j + 1)) * 8 for j in range(N // B))
    c2 = sum((M - B * j) * (N - B * (j + 1)) * 8 for j in range(1, N // B, 2))
    return {"gemm_tn": c + M * N * 8, "gemm_nn": 2 * c2}


def main(src, dst):
    rows = [r for r in csv.DictReader(l for l in open(src) if l.startswith('"'))]
    acc = collections.defaultdict(lambda: collections.defaultdict(float))
    ids = collections.defaultdict(set)
    for r in rows:
        k = r["Kernel Name"].split("(")[0].split("<")[0].replace("void ", "").split("::")[-1]
        k = k.replace("_kernel", "")
        acc[k][r["Metric Name"]] += float(r["Metric Value"].replace(",", ""))
        ids[k].add(r["ID"])
    alg = algorithmic_bytes()
    out = {"source": src.split("/")[-1], "workload": "C5 rqrcp 32768^2 b=128, one step, ncu --clock-control none"}
    for k, v in acc.items():
        n = len(ids[k])
        tot = v["dram__bytes_read.sum"] + v["dram__bytes_write.sum"]
        e = {"launches": n, "bytes_per_launch": tot / n, "read_bytes": v["dram__bytes_read.sum"],
             "write_bytes": v["dram__bytes_write.sum"], "ncu_ms_total": v["gpu__time_duration.sum"] / 1e6}
        if k in alg:
            e["algorithmic_bytes_per_launch"] = alg[k] / n
            e["traffic_over_algorithmic"] = tot / alg[k]
        out[k] = e
    json.dump(out, open(dst, "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
