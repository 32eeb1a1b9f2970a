#!/bin/bash
# Build libsbr.so + the oracle from any cwd; prints only errors.
cd "$(dirname "$0")/.." && python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -i -B2 -A2 "error" | head -30; ls -la paper_2504_21719_b200/_lib/libsbr.so | awk '{print $6, $7, $8, $9}'
