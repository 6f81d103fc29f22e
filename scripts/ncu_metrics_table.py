import csv,sys
def load(fn):
    rows=[r for r in csv.reader(open(fn)) if len(r)>10]
    hdr=rows[0]; idx={h:i for i,h in enumerate(hdr)}
    out={}
    for r in rows[1:]:
        k=int(r[idx['ID']]); out.setdefault(k,{'name':r[idx['Kernel Name']][:36]})
        out[k][r[idx['Metric Name']]]=float(r[idx['Metric Value']].replace(',',''))
    return out
fs=sys.argv[1:]
ds=[load(f) for f in fs]
for k in sorted(ds[0]):
    s=f"{k:2d} {ds[0][k]['name']:36s}"
    for d in ds:
        m=d.get(k,{})
        if not m: continue
        t=m['gpu__time_duration.sum']/1e3; tc=m['sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed']; l2=m['lts__t_bytes.sum']/1e6
        s+=f" | {t:6.1f}us tc{tc:5.1f}% L2 {l2:6.0f}MB {l2/t:5.1f}TB/s"
    print(s)
