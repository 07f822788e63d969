"""Stall samples per CUDA source line of an ncu report (tuning aid).

    ncu -i REPORT --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_lines.py src.csv [top]
"""
import csv, collections, sys
rows=list(csv.reader(open(sys.argv[1])))
hdr=rows[2]; iS=hdr.index("Warp Stall Sampling (All Samples)"); iE=hdr.index("Instructions Executed")
iW=hdr.index("L1 Wavefronts Shared")
src_line=None; agg=collections.Counter(); inst=collections.Counter(); wf=collections.Counter(); text={}
fname=""
for r in rows:
    if not r: continue
    if r[0] in ("File Path",): fname=r[1].split('/')[-1]; continue
    if r[0] in ("Function Name","Line No"): continue
    if len(r)<=iS: continue
    if r[0]:
        try: src_line=(fname,int(r[0])); text[src_line]=r[1].strip()
        except ValueError: continue
    try:
        agg[src_line]+=int(r[iS] or 0); inst[src_line]+=int(r[iE] or 0); wf[src_line]+=int(float(r[iW] or 0))
    except ValueError: pass
tot=sum(agg.values()); print("samples",tot,"inst",sum(inst.values()),"smem wavefronts",sum(wf.values()))
for l,s in agg.most_common(int(sys.argv[2]) if len(sys.argv)>2 else 45): print(f"{l[0][:12]}:{l[1]:<5} {s:5} {100*s/tot:5.1f}% inst {inst[l]:9} wf {wf[l]:9}  {text.get(l,'')[:80]}")
