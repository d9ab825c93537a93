"""Warp-stall samples of an ncu report per CUDA source line (developer tool).

    python scripts/ncu_source_lines.py REPORT.ncu-rep OUT.txt TITLE
"""
import csv,collections,sys,subprocess
rep, out_path, title = sys.argv[1], sys.argv[2], sys.argv[3]
raw=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(raw.splitlines()))
h=rows[2]; names=h[32:49]
f=None; agg=collections.Counter(); text={}; reasons=collections.defaultdict(collections.Counter)
tot=0
for r in rows:
    if len(r)>=2 and r[0]=='File Path': f=r[1].split('/')[-1]; continue
    if len(r)>=49 and r[0].isdigit():
        try: v=float(r[4])
        except: continue
        key=(f,int(r[0])); agg[key]+=v; tot+=v
        if r[1]: text[key]=r[1]
        for i in range(17):
            try: reasons[key][names[i]]+=float(r[32+i] or 0)
            except: pass
out=open(out_path,'w')
out.write(title+"\n"+f"total samples {tot:.0f}\n")
for (fn,l),v in agg.most_common(30):
    top=", ".join(f"{k[6:]}={int(x)}" for k,x in reasons[(fn,l)].most_common(3))
    out.write(f"{v:7.0f} {100*v/tot:5.1f}% {fn}:{l:<4} {text.get((fn,l),'')[:70]:70s} | {top}\n")
