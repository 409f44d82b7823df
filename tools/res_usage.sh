#!/bin/bash
# res_usage.sh LIB PATTERN: registers / stack per kernel whose name matches PATTERN
cuobjdump -res-usage "$1" 2>/dev/null | awk -v pat="$2" '/Function/ {name=$2} /REG:/ {if (name ~ pat) {match($0, /REG:[0-9]+/); r=substr($0, RSTART, RLENGTH); match($0, /STACK:[0-9]+/); s=substr($0, RSTART, RLENGTH); print r, s, name}}' | c++filt | sed -E 's/\(ismgb::fz::Params.*//'
