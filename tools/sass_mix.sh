#!/bin/bash
# opcode histogram of one kernel's SASS: tools/sass_mix.sh <object> <mangled-substring>
obj=$1; pat=$2
fn=$(cuobjdump -sass $obj | grep -o "Function : [^ ]*$pat[^ ]*" | head -1 | awk '{print $3}')
cuobjdump -sass -fun "$fn" $obj | grep -E "^\s+/\*[0-9a-f]+\*/" | sed 's/ *\/\* *0x[0-9a-f]* *\*\///' | sed 's/^ *\/\*[0-9a-f]*\*\/ *//' | sed 's/^@!*U*P[0-9T] *//' | awk '{print $1}' | sort | uniq -c | sort -rn | head -${3:-25}
