import csv, collections, sys
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == 'ID':
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d['Kernel Name'].split('(')[0].replace('asdsm_b200::<unnamed>::', '')[:60]
        v = float(d['Metric Value'].replace(',', ''))
        u = d['Metric Unit']
        v = v / 1e3 if u in ('nsecond', 'ns') else v * 1e3 if u in ('msecond', 'ms') else v
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"== {path}: {len(data)} launches, {tot/1e3:.2f} ms total (serialized)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:14]:
        print(f"  {v[1]:10.1f} us {100*v[1]/tot:5.1f}%  n={v[0]:4d}  {k}")
