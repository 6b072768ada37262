#!/bin/bash
for d in 0 1 2 3; do TCBF_DEBUG=$d VARIANTS=${VARIANTS:-1} python tools/sweep_f16.py ${1:-radio} 2>&1 | grep " v" | sed "s/^/debug=$d /"; done
