#!/bin/bash
# ncu --set full of one §5.1 in-place sequence launch (depth ${DEPTH:-16}, 56^2 unless H set)
O=gpurun_out/${TAG:-ncuseq}
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:seq_ -c 1 -o /tmp/seq -f \
     python scripts/prof_sec51.py ${DEPTH:-16} 0 2 > $O/ncu.log 2>&1
$NCU -i /tmp/seq.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
$NCU -i /tmp/seq.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
$NCU -i /tmp/seq.ncu-rep --page source --csv --print-source sass > $O/sass.csv 2>/dev/null
cp /tmp/seq.ncu-rep $O/
ls -la $O
