# K3 shape thresholds for mid-size calls: batch kernel from 16 slots (bm16), split rays up to 64k rays (sp64), both
for rep in 1 2; do for lib in libvxm.so libvxm_bm16.so libvxm_sp64.so libvxm_bm16sp64.so; do
  echo "== $lib"
  VXM_LIB_NAME=$lib QT_CONFIGS="cfg2:2,cfg2:4,cfg2:8,cfg2:12,cfg1:2,cfg1:4,cfg1:8,cfg1:12,cfg3:1,cfg3:2,cfg2:64" timeout 600 python tools/quick_time.py 2>&1 | grep graph
done; done > gpurun_out/r02cg_ab.txt 2>&1
cat gpurun_out/r02cg_ab.txt
