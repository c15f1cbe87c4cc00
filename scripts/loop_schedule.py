"""SASS check of the decode kernel's hot loop: length, positions of the ring-refill
LDG loads, spills.  usage: python scripts/loop_schedule.py <lib.so> [kernel-name-substring] [a:b]"""
import re,sys,subprocess,collections
lib=sys.argv[1]; pat=sys.argv[2] if len(sys.argv)>2 else 'decode_partials_m64b8ILb1ELb0ELi1ELi16'
fns=subprocess.run(['cuobjdump','-sass',lib],capture_output=True,text=True).stdout
fn=[l.split()[2] for l in fns.splitlines() if 'Function :' in l and pat in l][0]
txt=subprocess.run(['cuobjdump','-sass','-fun',fn,lib],capture_output=True,text=True).stdout
addr=[]
for l in txt.splitlines():
    m=re.match(r'\s*/\*([0-9a-f]+)\*/\s+(.*?)\s*;',l)
    if m: addr.append((int(m.group(1),16),m.group(2)))
best=None
for a,ins in addr:
    m=re.search(r'BRA.*?(0x[0-9a-f]+)',ins)
    if m and int(m.group(1),16)<a:
        t=int(m.group(1),16); body=[x for x in addr if t<=x[0]<=a]
        if sum('LDS' in x[1] for x in body)>=64 and (best is None or len(body)<len(best)): best=body
print(lib.split('/')[-1], 'loop', len(best), 'LDG at', [i for i,x in enumerate(best) if 'LDG' in x[1]], 'spills', sum('LDL' in x[1] or 'STL' in x[1] for x in addr))
if len(sys.argv)>3:
    a,b=map(int,sys.argv[3].split(':'))
    for i,x in enumerate(best[a:b]): print(a+i, x[1][:80])
