"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list per kernel name."""
import collections
import csv
import re
import sys


def summarize(path, steps=1, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    tot, cnt = collections.OrderedDict(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = re.sub(r'\(.*', '', r[ki]).split('::')[-1][:60]
        v = float(r[vi].replace(',', ''))
        tot[name] = tot.get(name, 0) + v
        cnt[name] += 1
    T = sum(tot.values())
    out = []
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:top]:
        out.append(f"{k:60s} {cnt[k] / steps:8.1f} {v / 1e6 / steps:9.3f} ms/step {100 * v / T:5.1f}%")
    out.append(f"total {T / 1e6 / steps:.3f} ms/step over {sum(cnt.values()) / steps:.0f} launches/step (serialised, cold-cache)")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1))
