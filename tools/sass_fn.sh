#!/bin/bash
# usage: tools/sass_fn.sh <lib> <function-substring>   -- print the SASS of the first matching function
cuobjdump -sass "$1" | awk -v pat="$2" '/Function : /{p = index($0, pat) > 0 && !done; if (p) done=1} p' | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed -E 's@ +/\* 0x[0-9a-f]+ \*/@@'
