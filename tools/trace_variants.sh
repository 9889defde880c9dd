#!/bin/bash
# Scratch: per-stage device times for trace-kernel variants (VXM_TRACE_VARIANT
# bit0 dedup, bit1 no atomics, bit2 no occupancy loads, bit3 lean loop).
for v in ${VARIANTS:-1 9}; do echo "variant $v"; VXM_TRACE_VARIANT=$v python tools/quick_time.py 2>&1; done
