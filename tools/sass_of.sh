#!/bin/bash
# usage: tools/sass_of.sh kernels.o out.sass  -- disassemble (with line info) the sm_100a cubin of an object
set -e
d=$(mktemp -d)
cp "$1" "$d/k.o"
(cd "$d" && cuobjdump -xelf all k.o > /dev/null)
nvdisasm -gi "$d"/*.cubin > "$2"
rm -rf "$d"
