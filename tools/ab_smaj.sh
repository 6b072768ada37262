#!/bin/bash
# Ablations of the radio fused fp16 kernels (dev build): which stream paces the tile loop.
# TCBF_DEBUG bits: 1 no output stores, 2 no MMAs, 4 no data reads, 8 weights once per unit
export AB_DEV_LIB=1 AB_REPS=${AB_REPS:-2}
AB_VARIANTS=${AB_VARIANTS:-"full:,noweights:TCBF_DEBUG=8,nostore:TCBF_DEBUG=1,nostore_now:TCBF_DEBUG=9,store_only:TCBF_DEBUG=6,store_only_now:TCBF_DEBUG=14,mma_only:TCBF_DEBUG=5,mc0:TCBF_F16_MC=0"} \
  python tools/ab_fused.py 1024 1024 256 256 ${AB_ITERS:-1500}
