#!/bin/bash
# Scratch: quick_time for each "LIBNAME:VARIANT" pair given in $AB
for ab in ${AB:-libvxm.so:1 libvxm.so:9}; do
  lib=${ab%%:*}; var=${ab##*:}
  echo "== $lib variant $var"
  VXM_LIB_NAME=$lib VXM_TRACE_VARIANT=$var python tools/quick_time.py 2>&1 | grep -A1 x64
done
