"""Per-kernel-class totals of an ncu launch list (gpu__time_duration.sum CSV)."""
import collections
import csv
import re
import sys


def kname(full: str) -> str:
    head = full.split("(")[0]
    while head.endswith(">"):  # strip trailing template arguments
        depth, i = 0, len(head) - 1
        for i in range(len(head) - 1, -1, -1):
            depth += head[i] == ">"
            depth -= head[i] == "<"
            if depth == 0:
                break
        head = head[:i]
    return re.split(r"::|\s", head)[-1]


def main(src, dst, title):
    rows = [r for r in csv.DictReader(l for l in open(src) if l.startswith('"'))]
    acc = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = kname(r["Kernel Name"])
        acc[k][0] += 1
        acc[k][1] += float(r["Metric Value"].replace(",", "")) / 1e6
    tot = sum(v[1] for v in acc.values())
    n = sum(v[0] for v in acc.values())
    lines = [title, f"launches {n}  total {tot:.1f} ms (serialised, cold-cache per launch)"]
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{k:36s} {v[0]:5d} {v[1]:9.1f} ms {100 * v[1] / tot:5.1f}%")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "ncu launch list")
