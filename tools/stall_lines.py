# Per-source-line stall samples of an ncu source page (--page source --csv --print-source sass), mapped with nvdisasm -g line info.
# usage: python tools/stall_lines.py page.csv <mangled kernel substring> [top]   (expects /tmp/elf/lines_cur.txt from nvdisasm -g -c)
import csv,re,collections,sys
rep=sys.argv[1]; fn=sys.argv[2]
lines=open('/tmp/elf/lines_cur.txt').read().splitlines()
st=[i for i,l in enumerate(lines) if l.startswith('//---') and fn in l][0]
cur=None; amap={}; sass={}
for l in lines[st+1:]:
    if l.startswith('//---') and '.text.' in l: break
    m=re.search(r'//## File "([^"]+)", line (\d+)',l)
    if m: cur=(m.group(1).split('/')[-1],int(m.group(2))); continue
    m=re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+([^;]*);',l)
    if m and cur: amap[int(m.group(1),16)]=cur; sass[int(m.group(1),16)]=m.group(2).strip()
rows=list(csv.reader(open(rep)))
hdr=rows[1]; data=rows[2:]
ia=hdr.index("Address"); iss=hdr.index("Warp Stall Sampling (All Samples)"); iex=hdr.index("Instructions Executed"); isrc=hdr.index("Source")
base=int(data[0][ia],16)
mism=sum(1 for r in data if (int(r[ia],16)-base) in sass and sass[int(r[ia],16)-base].split()[0] != r[isrc].strip().split()[0])
by=collections.defaultdict(lambda:[0,0]); tot=0; totx=0
for r in data:
    off=int(r[ia],16)-base; s=int(r[iss] or 0); e=int(r[iex] or 0)
    k=amap.get(off,('?',0)); by[k][0]+=s; by[k][1]+=e; tot+=s; totx+=e
print("mismatch",mism,"total samples",tot,"inst",totx)
src={f:open("/root/repo/paper_2106_02045_b200/csrc/"+f).read().splitlines() for f in ("sf_device.cuh","sf_fit_kernel.cuh","sf_init_core.cuh","sf_init.cu","sf_fit2l.cuh")}
for k,(s,e) in sorted(by.items(), key=lambda x:-x[1][0])[:int(sys.argv[3]) if len(sys.argv)>3 else 40]:
    t=src.get(k[0],[''])[k[1]-1].strip()[:70] if k[0] in src and k[1]>0 else ''
    print(f"{k[0][:14]:14s}:{k[1]:5d} {100*s/tot:5.1f}% samp {100*e/totx:5.1f}% inst  {t}")
