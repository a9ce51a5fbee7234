"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv): share per kernel."""
import collections, csv, sys

def main(path):
    rows = list(csv.DictReader(l for l in open(path) if not l.startswith('==')))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r['Metric Name'] != 'gpu__time_duration.sum':
            continue
        v = float(r['Metric Value'])
        u = r['Metric Unit']
        v = v / 1e3 if u in ('ns', 'nsecond') else v * 1e3 if u in ('ms', 'msecond') else v  # -> us
        name = r['Kernel Name'].split('(')[0][:48] + ' ' + r['Grid Size']
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v for _, v in agg.values())
    for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{v / tot * 100:5.1f}%  n={n:3d}  avg={v / n:9.1f} us  {k}")
    print(f"total {tot / 1e3:.2f} ms over {sum(n for n, _ in agg.values())} launches")

if __name__ == '__main__':
    main(sys.argv[1])
