#!/bin/bash
# c64 tile-pass knobs on sup32 / var20 (prefetch depth, CTAs per SM, CTA pairs, ring)
mkdir -p gpurun_out/c64k
QJ_AB="${QJ_AB2:-base:}" \
QJ_WL="${QJ_WL2:-sup32_c64}" bash tools/ab_tile.sh 2>&1 | python3 -c "
import sys,json
for l in sys.stdin:
    parts=l.split(); j=l[l.find('{'):]
    try:
        d=json.loads(j); print(parts[0], parts[1], 'sim %.4f'%d['simulate'], 'sep %.4f'%d['separate'])
    except Exception as e: print(l[:300])
" | tee gpurun_out/c64k/summary.txt
