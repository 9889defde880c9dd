// Single translation unit for libvxm.so: the kernels are header-defined
// templates of one module, so the runtime and the stage entry points are
// compiled together (one copy of every __global__ function in the cubin).
#include "vxm_runtime.cu"
#include "vxm_stages.cu"
