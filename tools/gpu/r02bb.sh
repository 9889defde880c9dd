for rep in 1 2; do for lib in libvxm.so libvxm_sq5.so libvxm_sq6.so; do
  echo "== $lib"; VXM_LIB_NAME=$lib QT_CONFIGS="cfg1:1:64,cfg2:1:64" timeout 300 python tools/quick_time.py 2>&1 | grep -A1 graph
done; done
