/*
 * rsim_bench.h -- measurement helpers shipped in librsim.so (not part of the
 * reference-facing ABI in rsim.h).
 */
#ifndef RSIM_BENCH_H
#define RSIM_BENCH_H
#ifdef __cplusplus
extern "C" {
#endif

/* Sustained FMA throughput of the FP64 (fp64=1) or FP32 (fp64=0) pipe on the
 * current device, in TFLOP/s (2 flops per FMA).  Returns 0 on success. */
int rsim_bench_fma_peak(int fp64, double *tflops);

/* Executed-work calibration of the renderer: one render launch of cam_mask
 * (no image writes) that atomically adds the number of ray-plane tests
 * (sphere test = 1) it executed to *d_counter (device uint64). */
struct rs_batch;
int rsim_bench_render_work(struct rs_batch *batch, unsigned int cam_mask, unsigned long long *d_counter,
                           void *stream);
/* same for rs_render_mesh: counts candidate-part BVH traversals */
int rsim_bench_render_mesh_work(struct rs_batch *batch, unsigned int cam_mask, unsigned long long *d_counter,
                                void *stream);

#ifdef __cplusplus
}
#endif
#endif
