#!/bin/bash
# usage: tools/spills.sh <mangled-kernel-substring>  -- spill sites by source line in libnsdgt.so
set -e
d=$(mktemp -d); cd $d
cuobjdump -xelf all /root/repo/paper_1307_4569_b200/libnsdgt.so >/dev/null 2>&1
nvdisasm -g -c dgt.sm_100a.cubin 2>/dev/null | awk -v k="$1" '$0 ~ "\\.text\\..*"k {f=1;next} /\.text\./{if(f)exit} f' > k.sass
python3 - <<'PY'
import re, collections
lines=open('k.sass').read().split('\n')
hist=[]; out=[]
for l in lines:
    m=re.search(r'//## File "([^"]+)", line (\d+)',l)
    if m: hist.append(m.group(1).split('/')[-1]+':'+m.group(2)); continue
    if 'STL' in l or 'LDL' in l:
        ctx=[h for h in hist[-80:] if 'fused7' in h and int(h.split(':')[1])>200]
        out.append(('STL' if 'STL' in l else 'LDL', ctx[-1] if ctx else None))
for k,v in collections.Counter(out).most_common(20): print(v,k)
PY
rm -rf $d
