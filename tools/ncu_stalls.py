"""Stall reasons, instruction mix and the top stalled SASS lines from `ncu --page source --csv --print-source sass` output: python tools/ncu_stalls.py sass.csv [top]."""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[1]; idx={h:i for i,h in enumerate(hdr)}
def f(x):
    try: return float(x or 0)
    except ValueError: return None
S="Warp Stall Sampling (All Samples)"; IE="Instructions Executed"
data=[r for r in rows[2:] if len(r)==len(hdr) and f(r[idx[S]]) is not None]
seen=set(); d2=[]
for r in data:
    if r[0] in seen: continue
    seen.add(r[0]); d2.append(r)
data=d2
tot=sum(f(r[idx[S]]) for r in data); ti=sum(f(r[idx[IE]]) for r in data)
st=[h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg={h:sum(f(r[idx[h]]) for r in data) for h in st}
print("total stall",tot,"instr",ti); print(sorted(((round(v/tot*100,1),k[6:]) for k,v in agg.items()),reverse=True)[:9])
mix=collections.Counter()
for r in data:
    t=r[1].split(); op=t[1] if t[0].startswith('@') else t[0]
    mix[op.split('.')[0]]+=f(r[idx[IE]])
print([(k, round(v/ti*100,1)) for k,v in mix.most_common(22)])
top=sorted(data, key=lambda r:-f(r[idx[S]]))[:int(sys.argv[2]) if len(sys.argv)>2 else 14]
for r in top:
    s=f(r[idx[S]])
    reasons=sorted(((f(r[idx[h]]),h) for h in st),reverse=True)[:2]
    print(f"{r[0][-5:]} {s/tot*100:5.1f}% {r[1][:60]:60s} {[(int(a),b[6:]) for a,b in reasons]}")
