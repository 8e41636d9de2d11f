import csv,sys,glob,collections
for f in sorted(glob.glob(sys.argv[1])):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    if not rows: print(f,"empty"); continue
    h=rows[0]; data=rows[1:]
    iK=h.index("Kernel Name"); iM=h.index("Metric Name"); iV=h.index("Metric Value"); iI=h.index("ID")
    per=collections.defaultdict(dict); name={}
    for r in data:
        if r[iM] in ("Metric Name",): continue
        per[r[iI]][r[iM]]=r[iV]; name[r[iI]]=r[iK]
    agg=collections.defaultdict(list)
    for i,m in per.items():
        k=name[i].split("(")[0].replace("void tc::tc_gemm_kernel","")
        agg[k].append(m)
    tot=0
    out=[]
    for k,ms in agg.items():
        def av(key): 
            v=[float(m[key].replace(",","")) for m in ms if key in m]; return sum(v)/len(v) if v else float('nan')
        dur=av("gpu__time_duration.sum"); tot+=dur*len(ms)
        out.append(f"  {k:22s} n={len(ms)} dur={dur/1e3:8.1f}us clk={av('sm__cycles_elapsed.avg.per_second')/1e6:6.0f}MHz tens={av('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):5.1f}% rd={av('dram__bytes_read.sum')/1e9 if 'dram__bytes_read.sum' in ms[0] else 0:.2f}")
    print(f, f"total/step={tot/1e3/ (len(data) and 2):.0f}us")
    print("\n".join(out))
