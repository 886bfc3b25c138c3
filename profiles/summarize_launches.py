import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hi]; data = rows[hi+1:]
kn = hdr.index('Kernel Name'); mv = hdr.index('Metric Value'); mn = hdr.index('Metric Name')
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in data:
    if r[mn] != 'gpu__time_duration.sum': continue
    name = r[kn].split('(')[0]
    v = float(r[mv].replace(',',''))
    tot[name] += v; cnt[name] += 1
T = sum(tot.values())
for k,v in sorted(tot.items(), key=lambda x:-x[1])[:int(sys.argv[2]) if len(sys.argv)>2 else 20]:
    print(f"{k:50s} n={cnt[k]:6d} total={v/1e6:9.3f} ms share={v/T:6.1%} avg={v/cnt[k]/1e3:8.2f} us")
print('total ms', T/1e6)
