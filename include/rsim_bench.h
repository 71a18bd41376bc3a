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
/* The same launch with the 20 counters of the counting variant (added to
 * d_counters[20], device uint64): 0 FP32 box plane tests, 1 FP64 plane tests
 * in the walk (uncertain boxes, hulls; sphere = 1), 2 FP64 plane tests
 * resolving candidates, 3 pixels that fell back to the all-FP64 walk,
 * 4 uncertain boxes, 5 hull tests in the walk, 6 plane tests of the all-FP64
 * walk, 7 pixels, 8 FP32 box tests that missed, 9 hits that did not become
 * candidates, 10 tile-list entries visited, 11 entries outside the part's
 * pixel rectangle; SM cycles summed over CTAs: 12 camera pose, 13 part
 * frames, 14 world planes, 15 culling + ordering, 16 tile lists, 17 trace;
 * summed over warps: 18 culling warps' own work, 19 ordering warps'. */
int rsim_bench_render_work_detail(struct rs_batch *batch, unsigned int cam_mask, unsigned long long *d_counters,
                                  void *stream);
/* rs_render with every ray test in FP64 (rs_render selects candidates with
 * bounded-error FP32 box tests and resolves them in FP64; this variant is its
 * parity reference). Same arguments and outputs as rs_render. */
int rsim_bench_render_exact(struct rs_batch *batch, unsigned int cam_mask, unsigned char *rgba, float *depth,
                            int *ids, void *stream);
/* Per-env step latency probe: when d_cycles (device int64[E]) is set, every
 * step writes each env's SM clock cycles from kernel entry to its state
 * write-back (negated for envs run by the contact-heavy CTA kernel); NULL
 * turns the probe off. */
int rsim_bench_env_cycles(struct rs_batch *batch, long long *d_cycles);
/* Per-env phase clock accumulators (device int64 [n_env][16], added to by
 * every warp-per-env step; NULL = off): 0 substep front (kinematics, broad-
 * and narrowphase, rows), 1 Gauss-Seidel sweeps, 2 eigensolves, 3 block LCP
 * iterations, 4 block impulse + friction, 5 scalar rows, 6 integrate/joints;
 * the front split into 7 kinematics, 8 AABBs + overlap, 9 admission,
 * 10 narrowphase, 11 rows + blocks. */
int rsim_bench_phase_cycles(struct rs_batch *batch, long long *d_cycles);
/* Debug scheduling hook (parity tests): width 8 or 16 = every env of the
 * following rs_step calls runs in the contact-heavy CTA kernel of that many
 * warps (wavefront Gauss-Seidel); -8 or -16 = the normal heavy-env
 * selection with CTAs of that width; 0 = the normal heavy-env scheduling. */
int rsim_bench_force_heavy(struct rs_batch *batch, int width);
/* same for rs_render_mesh: counts candidate-part BVH traversals */
int rsim_bench_render_mesh_work(struct rs_batch *batch, unsigned int cam_mask, unsigned long long *d_counter,
                                void *stream);

#ifdef __cplusplus
}
#endif
#endif
