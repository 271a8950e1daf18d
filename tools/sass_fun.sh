#!/bin/bash
# usage: tools/sass_fun.sh LIB.so MANGLED_NAME -- SASS of one function (instruction lines only)
cuobjdump -sass "$1" | awk -v f="$2" '/Function : /{on = ($3 == f)} on' | grep -E '^\s+/\*[0-9a-f]{4,6}\*/'
