#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over the C1 smoke layer
# (plan -> select -> sparse attention) on the GPU box. Round-1 result: 0 errors / 0 hazards.
for t in memcheck racecheck synccheck; do
  echo "== $t"
  timeout 400 compute-sanitizer --tool $t --print-limit 5 \
    python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | grep -E "SUMMARY|smoke ok|error detected|at fp"
done
