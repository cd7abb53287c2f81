#!/bin/bash
# usage: scripts/spill_lines.sh obj.o  -> source lines of local-memory (spill) instructions per kernel
cd /tmp && rm -rf spl && mkdir spl && cd spl && cuobjdump -xelf all "$1" >/dev/null 2>&1
for c in *.cubin; do nvdisasm -g -c "$c" 2>/dev/null; done | awk '/\.text\./{fn=$0} /line [0-9]+/{match($0,/line [0-9]+/); ln=substr($0,RSTART,RLENGTH)} /(STL|LDL)/{print fn" "ln}' | sort | uniq -c | sort -rn | head -${2:-15}
