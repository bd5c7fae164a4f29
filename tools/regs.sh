#!/bin/bash
# registers / spills of the main 4096/2048 instantiations, from the nvcc -Xptxas -v logs
cd /root/repo/paper_2008_12214_b200/csrc/build
for f in k_row k_col_gs k_col_gsg k_col_ospr k_col_plain; do
  grep -E "Compiling entry|registers|spill" $f.o.log | paste - - - 2>/dev/null | \
  python3 -c "
import sys,re
for l in sys.stdin:
    n=re.search(r\"function '_ZN2hg5(k_\w+?)EEEvNS\",l); s=re.search(r'(\d+) bytes spill stores',l); r=re.search(r'Used (\d+) registers',l)
    if n and r and re.search(r'ILi(4096|2048)E',n.group(1)): print(n.group(1), 'regs', r.group(1), 'spill', s.group(1) if s else '?')
"
done
