# cfg4 trajectory A/B: r02bm build (bm), + pointer slabs/lane counts/prologue (pro), + chain publish (pub), HEAD (libvxm)
for rep in 1 2; do for lib in libvxm_bm.so libvxm_pro.so libvxm_pub.so libvxm.so; do
  echo "== $lib $(VXM_LIB_NAME=$lib timeout 300 python tools/probes/traj_probe.py 2>&1 | tail -1)"
done; done > gpurun_out/r02bw_traj.txt 2>&1
cat gpurun_out/r02bw_traj.txt
