/*
 * ORACLE / TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference
 * voxmap per-frame path (Sequential mode), used by tests/ and bench.py's
 * CPU-baseline leg as the checker. Never linked into the product.
 *
 * Pinned: tests/test_cpu_oracle.py checks it byte for byte against the
 * reference's own sources compiled here (oracle/_ref) and against the
 * committed golden vectors in tests/golden/ (made by tests/golden/make_golden.py
 * from the reference build), including the reference's known-answer tests.
 *
 * Structs are the vxm.h PODs. Grids are uint8 arrays, idx = x + y*dx + z*dx*dy.
 */
#ifndef VOXMAP_ORACLE_H_
#define VOXMAP_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#include "../include/vxm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* kernels_scalar.cpp:10-16 */
void vo_merge(uint8_t* local, const uint8_t* ms, size_t n);
/* kernels_scalar.cpp:18-37 (R row-major) */
void vo_transform_voxelize(const double* xs, const double* ys, const double* zs, size_t n,
                           const double* R, const double* t, double vs, int32_t* cx,
                           int32_t* cy, int32_t* cz);
/* geometry.cpp:43-99 (Sequential); returns the point count, -1 on bad camera */
long long vo_depth_to_cloud(const vxm_camera* cam, const float* depth, double* xs, double* ys,
                            double* zs);
/* integrator.cpp:45-103 */
int vo_populate(const vxm_grid_spec* g, uint8_t* ms, const double* xs, const double* ys,
                const double* zs, size_t n, const vxm_pose* t_vc, int vox_inf,
                vxm_populate_stats* st);
/* raytracer.cpp:8-21 */
int vo_bundle_dimensions(const vxm_camera* cam, double depth, double vs, int32_t out[3]);
/* raytracer.cpp:35-118 + raytracer.hpp:76-118 (Sequential) */
int vo_trace_bundle(const vxm_grid_spec* g, uint8_t* ms, const int32_t bundle[3],
                    const vxm_pose* t_vc, vxm_trace_stats* st);
/* raytracer.hpp:136-194 + raytracer.cpp:120-161 (Sequential) */
int vo_trace_per_pixel(const vxm_grid_spec* g, uint8_t* ms, const double* xs, const double* ys,
                       const double* zs, size_t n, const vxm_pose* t_vc, vxm_trace_stats* st);
/* grid.cpp:81-108 */
void vo_shift(const int32_t dims[3], const uint8_t* in, uint8_t* out, const int32_t off[3]);

/* MappingPipeline (pipeline.cpp:68-117), Sequential. */
typedef struct vo_pipeline vo_pipeline;
vo_pipeline* vo_pipeline_create(const vxm_config* cfg);
void vo_pipeline_destroy(vo_pipeline* p);
int vo_pipeline_integrate_cloud(vo_pipeline* p, const double* xs, const double* ys,
                                const double* zs, size_t n, const vxm_pose* t_wc, vxm_stats* st);
int vo_pipeline_integrate_depth(vo_pipeline* p, const float* depth, const vxm_pose* t_wc,
                                vxm_stats* st);
void vo_pipeline_local(const vo_pipeline* p, uint8_t* cells, double origin[3]);

#ifdef __cplusplus
}
#endif

#endif
