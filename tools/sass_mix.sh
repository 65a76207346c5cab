#!/bin/bash
# Opcode histogram of one kernel's SASS: tools/sass_mix.sh <object/.so> <mangled-name-regex>
obj=$1; pat=$2
fn=$(cuobjdump -sass "$obj" | grep -oE "Function : [^ ]+" | awk '{print $3}' | grep -E "$pat" | head -1)
cuobjdump -sass -fun "$fn" "$obj" | grep -E "^\s+/\*[0-9a-f]{4,}\*/" | sed -E 's#^\s+/\*[0-9a-f]+\*/\s+##; s#^@!?U?P[T0-9]+\s+##' | awk '{print $1}' | sed 's/\..*//;s/;//' | sort | uniq -c | sort -rn | head -${3:-25}
echo "function: $fn"
