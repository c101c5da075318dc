"""Summarise per-rank device timelines written by bench.py under DK_TRACE_TS=1.

    python tools/ts_analyze.py ts_cg_n4.json

Per interval between consecutive marks: the median over iterations on each rank (globaltimer
clocks are per GPU, so only intervals within one rank are compared), plus the iteration period.
"""

import collections
import json
import statistics
import sys


def main(path):
    d = json.load(open(path))
    W = len(d)
    labels = [lab for lab, _ in d[0]]
    first = labels[0]
    starts = [i for i, lab in enumerate(labels) if lab == first]
    per = collections.defaultdict(lambda: [[] for _ in range(W)])
    for k in range(len(starts) - 1):
        a, b = starts[k], starts[k + 1]
        seen = collections.Counter()
        for i in range(a, b):
            key = f"{labels[i]} -> {labels[i + 1]}"
            seen[key] += 1
            if seen[key] > 1:
                key += f" #{seen[key]}"
            for r in range(W):
                per[key][r].append((d[r][i + 1][1] - d[r][i][1]) / 1e3)
        for r in range(W):
            per["PERIOD"][r].append((d[r][b][1] - d[r][a][1]) / 1e3)
    print(f"{'interval (us, median per rank)':64s}" + "".join(f"{'r' + str(r):>9s}" for r in range(W)))
    for key, v in per.items():
        print(f"{key[:64]:64s}" + "".join(f"{statistics.median(x):9.1f}" for x in v))
    print("PERIOD per iteration, rank 0:", [round(x) for x in per["PERIOD"][0]])


if __name__ == "__main__":
    main(sys.argv[1])
