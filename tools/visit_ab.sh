#!/bin/bash
# nodes / triangles per ray-bounce: default (speculative) traversal vs -DSBR_NO_SPECULATE
# (build first: tools/build_variants.sh visits "-DSBR_COUNT_VISITS" visits_nospec "-DSBR_COUNT_VISITS -DSBR_NO_SPECULATE")
for v in visits visits_nospec; do SBR_VISITS_LIB=$v python tools/visit_stats.py | sed "s/^/$v /"; done
