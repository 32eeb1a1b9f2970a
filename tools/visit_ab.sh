#!/bin/bash
# nodes / triangles per ray-bounce: default traversal vs -DSBR_SPECULATE
# (build first: tools/build_variants.sh visits "-DSBR_COUNT_VISITS" visits_spec "-DSBR_COUNT_VISITS -DSBR_SPECULATE")
for v in visits visits_spec; do SBR_VISITS_LIB=$v python tools/visit_stats.py | sed "s/^/$v /"; done
