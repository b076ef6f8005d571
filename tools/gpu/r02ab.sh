mkdir -p gpurun_out
T=${T:-r02ab}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c4n127rk4.csv python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 30 > /dev/null 2>&1
python - <<'P'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/r02ab_launches_c4n127rk4.csv')) if r and not r[0].startswith('==')]
h=rows[0]; ix={k:i for i,k in enumerate(h)}
acc=collections.defaultdict(lambda:[0,0.0])
for r in rows[1:]:
    n=r[ix['Kernel Name']].split('(')[0]; t=float(r[ix['Metric Value']].replace(',',''))*1e-6
    acc[n][0]+=1; acc[n][1]+=t
tot=sum(v[1] for v in acc.values())
for k,v in sorted(acc.items(), key=lambda x:-x[1][1]): print(f"{k[:70]:70s} n={v[0]:5d} ms={v[1]:9.2f} share={v[1]/tot:.3f} avg={v[1]/v[0]:.3f}")
P
timeout 300 python tools/profile_case.py --config 4 --n-rods 127 --method rk4 --slices 30 | tail -2
