# Loop-body finder for cuobjdump -sass listings: prints each backward-branch loop with its instruction mix.
# usage: python tools/sass_loops.py listing.sass <first line of the function in the listing>
import re,sys,collections
lines=open(sys.argv[1]).read().splitlines()
start=int(sys.argv[2]); end=int(sys.argv[3]) if len(sys.argv)>3 else len(lines)
ins=[]
for l in lines[start:end]:
    m=re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);',l)
    if m: ins.append((int(m.group(1),16),m.group(2).strip()))
addr={a:i for i,(a,_) in enumerate(ins)}
for i,(a,t) in enumerate(ins):
    m=re.search(r'BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))',t)
    mm=re.search(r'BRA.*?0x([0-9a-f]+)',t)
    if mm:
        tgt=int(mm.group(1),16)
        if tgt<=a and tgt in addr:
            j=addr[tgt]; body=ins[j:i+1]
            c=collections.Counter()
            for _,x in body:
                x=re.sub(r'^@!?U?P\w+\s+','',x)
                op=x.split()[0]
                c[op.split('.')[0]]+=1
            print(f"loop {tgt:#x}-{a:#x}: {len(body)} instrs", dict(c.most_common(25)))
