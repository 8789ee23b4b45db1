#!/bin/bash
for d in 0 1 8 16 24; do echo "== NSB_DEBUG_BLOCKED=$d"; NSB_DEBUG_BLOCKED=$d python tools/tma_debug.py 1 2>&1 | grep -v "^   at"; done
echo "== promo none"; NSB_TMA_PROMO=0 python tools/tma_debug.py 1 2>&1 | grep -v "^   at"
