#!/bin/bash
# Build experiment libraries: each arg is "TILE:DEFS" (either part may be empty),
# e.g.  scripts/buildvars.sh "8x1:" "2x4:" "8x1:CCL_JUMP=0" ; prints the .so paths.
cd "$(dirname "$0")/.."
for spec in "$@"; do
  tile="${spec%%:*}"; defs="${spec#*:}"
  CCL_TILE="$tile" CCL_DEFS="$defs" python paper_1712_09789_b200/_build.py &
done
wait
