import csv, re, sys, subprocess, collections
rep, cubin, fn = sys.argv[1], sys.argv[2], sys.argv[3]
txt=subprocess.run(['nvdisasm','-g','-c',cubin],capture_output=True,text=True).stdout.split('\n')
start=[i for i,l in enumerate(txt) if l.startswith('//--------------------- .text.'+fn+' ')][0]
lmap={}; cur=None
for l in txt[start+1:]:
    if l.startswith('//--------------------- .text'): break
    m=re.search(r'File ".*/([^/"]+)", line (\d+)',l)
    if m: cur=(m.group(1),int(m.group(2))); continue
    m=re.match(r'\s+/\*([0-9a-f]{4,})\*/',l)
    if m: lmap[int(m.group(1),16)]=cur
out=subprocess.run(["ncu","-i",rep,"--page","source","--csv","--print-source","sass"],capture_output=True,text=True).stdout
rows=list(csv.reader(out.splitlines())); hdr=rows[1]; data=rows[2:]
ia=hdr.index('Address'); iss=hdr.index('Warp Stall Sampling (All Samples)'); iex=hdr.index('Instructions Executed')
reasons=[h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]; ri=[hdr.index(h) for h in reasons]
f=lambda v: float(v) if v not in ('',None,'-') else 0.0
a0=int(data[0][ia],16)
agg=collections.defaultdict(lambda: [0.0,0.0,collections.Counter()])
tot=0
for r in data:
    off=int(r[ia],16)-a0; key=lmap.get(off)
    s=f(r[iss]); tot+=s
    agg[key][0]+=s; agg[key][1]+=f(r[iex])
    for h,i in zip(reasons,ri): agg[key][2][h[6:]]+=f(r[i])
items=sorted(agg.items(), key=lambda kv:-kv[1][0])
for k,(s,ex,rs) in items[:int(sys.argv[4]) if len(sys.argv)>4 else 40]:
    print(f"{str(k):32s} {s/tot*100:5.1f}% inst={ex:.3g} | "+" ".join(f"{a}:{b/s*100:.0f}" for a,b in rs.most_common(4) if s>0))
