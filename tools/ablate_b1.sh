#!/bin/bash
for d in 0 1 2 4 3 5 6 7; do echo -n "debug=$d "; TCBF_DEBUG=$d python tools/quick_time.py ${1:-radio_b1} 2>&1 | tail -1 | cut -c1-110; done
