# Sum an ncu --csv launch list per kernel, from the last k_fold_keys launch on
# (= the second set_points of scripts/setpts_only.py).
import csv,sys
for v in sys.argv[1:]:
    print('==', v)
    rows=[r for r in csv.reader(open(v)) if len(r)>10]
    h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
    data=rows[1:]
    last=max(i for i,r in enumerate(data) if 'k_fold_keys' in r[ki])
    data=data[last:]
    tot={}; cnt={}
    for r in data:
        k=r[ki][:70]; tot[k]=tot.get(k,0)+float(r[vi].replace(',','')); cnt[k]=cnt.get(k,0)+1
    for k,x in sorted(tot.items(), key=lambda x:-x[1]): print('%9.1f us x%d'%(x/1e3,cnt[k]), k)
    print('total', sum(tot.values())/1e3)
