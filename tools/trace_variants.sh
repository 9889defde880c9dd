for v in 0 1 2 3 4; do echo "variant $v"; VXM_TRACE_VARIANT=$v python tools/quick_time.py 2>&1 | grep -v "^   " ; done
