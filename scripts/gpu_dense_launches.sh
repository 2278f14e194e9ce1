timeout 600 ncu --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio --clock-control none -k regex:dense_coef --csv --log-file gpurun_out/launches_9x500_dense.csv python scripts/profile_config.py mnist_9x500 1 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/launches_9x500_dense.csv')))
h=next(i for i,r in enumerate(rows) if 'Kernel Name' in r)
hdr=rows[h]; data=rows[h+1:]
ki=hdr.index('Kernel Name'); gi=hdr.index('Grid Size'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); idi=hdr.index('ID')
L=collections.defaultdict(dict)
for r in data:
    if len(r)<=vi: continue
    L[r[idi]]['k']=r[ki].split('(')[0]; L[r[idi]]['g']=r[gi]; L[r[idi]][r[mi]]=float(r[vi].replace(',',''))
for l in list(L.values())[-40:]:
    print(l['k'][:22], l['g'], {k.split('__')[1][:40]: round(v,2) for k,v in l.items() if '__' in k})
PY
