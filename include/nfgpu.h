/*
 * nfgpu.h — C ABI of the B200-native SPGM operator for near-field MIMO imaging.
 *
 * This is the drop-in boundary for the hot path of the reference package
 * `nfmimo` (arXiv 2509.00774). The reference has no FFI of its own. Its operator
 * "API" is a set of module-level Python functions. Each entry point below
 * replaces one of them, and the Python host package `paper_2509_00774_b200`
 * binds these symbols with ctypes (INTEGRATION.md shows the stub).
 *
 *   nf_plan_create        replaces  forward._plan / _OperatorPlan      pkg/src/nfmimo/forward.py:183-211
 *                                   (phasor tables F×(T+R)×N are NOT built; a frequency-free
 *                                    per-(antenna, voxel) distance table is built instead)
 *   nf_batch_prepare      replaces  forward._subset_indices + _channel_groups  forward.py:227-258
 *   nf_sample_structured  device counterpart of solver.sample_minibatch (solver.py:205-225)
 *   nf_batch_prepare_structured  replaces the same for the Cartesian subsets that
 *                                 solver.sample_minibatch draws (solver.py:205-225) and for the
 *                                 full channel set (forward.py:233-236); separable fast path
 *   nf_forward            replaces  forward.forward_apply / _forward_values    forward.py:342-350, 268-289
 *   nf_adjoint            replaces  forward.adjoint_apply / _adjoint_values    forward.py:353-359, 292-336
 *   nf_adjoint_prox       replaces  solver._gradient + soft_threshold +
 *                                   relative_magnitude_change (one SPGM step)  solver.py:181-183, 228-251, 287-289
 *   nf_spgm_loop          replaces  solver._solve's iteration loop for flat batches    solver.py:259-318
 *   nf_spgm_loop_chained            (K iterations per launch, device-side termination test)
 *   nf_sample_flat        replaces  host minibatch sampling (flat uniform w/o replacement; the
 *   nf_plan_set_iter                structured Cartesian sampler solver.py:206-225 stays on the host)
 *   nf_soft_threshold     replaces  solver.soft_threshold                      solver.py:228-241
 *   nf_magnitude_change   replaces  solver.relative_magnitude_change           solver.py:244-251
 *
 * Conventions (all match the reference):
 *   channel m = ri + R*(ti + T*fi)                       geometry.py:316-333
 *   voxel   n = ix + nx*(iy + ny*iz), x fastest           geometry.py:128-129
 *   A[m,n]  = p_f * exp(-j*2*pi*f*(dT+dR)/c) / (4*pi*dT*dR)   forward.py:142-155
 *   adjoint = sum_k conj(A[m_k,n]) * r_k                  forward.py:353-354
 *
 * Memory: every vector argument is a DEVICE pointer owned by the caller.
 * Complex vectors are interleaved (re, im) pairs of float (NF_C64) or double
 * (NF_C128). A plan covers the voxel z-slab [z_begin, z_end); voxel vectors
 * passed to a plan are indexed by the slab-local flat index
 * n - z_begin*nx*ny. Channel index lists are int32. All calls are
 * stream-ordered on `stream` (a cudaStream_t, NULL = legacy default stream);
 * one plan must be used from one stream at a time. Calls never throw.
 * They return NF_OK or a negative status, and nf_last_error() describes the failure.
 */
#ifndef NFGPU_H
#define NFGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NF_OK 0
#define NF_ERR_ARG -1     /* invalid argument (reference: ValueError) */
#define NF_ERR_RANGE -2   /* index out of range (reference: IndexError) */
#define NF_ERR_CUDA -3    /* CUDA runtime failure */
#define NF_ERR_STATE -4   /* call order violated (e.g. forward before batch_prepare) */

#define NF_C64 0  /* complex64 storage, fp32 entries with fp64 anchors (north star: rel L2 <= 1e-5) */
#define NF_C128 1 /* complex128 storage, fp64 everywhere (north star: rel L2 <= 1e-10) */

typedef struct nf_plan nf_plan;

/* Build a plan for one voxel slab. Host pointers:
 *   tx_xyz (n_tx*3), rx_xyz (n_rx*3)         antenna positions [m]      geometry.py:49-84
 *   freq_hz (n_f)                            np.linspace values         geometry.py:118-120
 *   pulse_reim (2*n_f)                       p(f) at each frequency     geometry.py:231-269
 *   corner[3], spacing[3], dims[3]           VoxelGrid corner/spacing/dims  geometry.py:157-166
 *   z_begin, z_end                           slab of z-planes owned by this plan (0, dims[2] = all)
 *   max_batch                                largest channel batch that will be prepared (<= M)
 * The distance table (8 or 16 bytes per antenna-voxel pair) is built on the current device. */
int nf_plan_create(const double* tx_xyz, int n_tx, const double* rx_xyz, int n_rx,
                   const double* freq_hz, const double* pulse_reim, int n_f, double c,
                   const double corner[3], const double spacing[3], const int dims[3],
                   int z_begin, int z_end, int dtype, int max_batch, nf_plan** out);
int nf_plan_destroy(nf_plan* plan);

/* info[0]=slab voxels, [1]=M, [2]=warp tiles, [3]=tx group size, [4]=device bytes held,
 * [5]=forward window (channels per forward launch), [6]=dtype, [7]=kernel launches issued so far */
int nf_plan_info(const nf_plan* plan, int64_t info[8]);

/* Stage a channel subset (device int32, length B, subset order, validated by the caller:
 * distinct, 0 <= m < M). Sorts it into the kernels' work order on the device. The staged
 * batch is used by every following forward/adjoint call until the next prepare. */
int nf_batch_prepare(nf_plan* plan, const int32_t* idx_dev, int batch, void* stream);

/* Stage the structured subset Fs × Ts × Rs (HOST int32 lists, each strictly increasing and
 * in range; validated here). Its channels m = r + R(t + T f) in lexicographic (f, t, r) order,
 * which is ascending m, form the subset order (batch = nf·nt·nr). The kernels then use the
 * factorisation A[(f,t,r), n] = p_f/(4π)·U_ft(n)·V_fr(n): n_t + n_r phasors per
 * (frequency, voxel) instead of n_t·n_r, and complex multiply-adds for the contraction.
 * Results equal nf_batch_prepare on the same channel list to within rounding. */
int nf_batch_prepare_structured(nf_plan* plan, const int32_t* fs, int nf, const int32_t* ts, int nt,
                                const int32_t* rs, int nr, void* stream);

/* y[k] = sum_{n in slab} A[m_k, n] s[n] for the staged batch, k in subset order. */
int nf_forward(nf_plan* plan, const void* s_dev, void* y_dev, void* stream);

/* g[n] = scale * sum_k conj(A[m_k, n]) (r[k] - ymeas[m_k]); ymeas may be NULL (treated as 0).
 * r is in subset order, ymeas is the full length-M measurement vector. */
int nf_adjoint(nf_plan* plan, const void* r_dev, const void* ymeas_dev, void* g_dev, double scale,
               void* stream);

/* Fused SPGM update over the slab:
 *   g = sum_k conj(A[m_k,n]) (r[k] - ymeas[m_k]);  u = s_in - eta_over_b * g;
 *   s_out = soft_threshold(u, alpha)            (solver.py:288, 228-241)
 * stats_dev (device, 4 doubles) receives {sum |s_in|^2, sum (|s_out|-|s_in|)^2,
 * (1/2) sum_k |r_k - ymeas[m_k]|^2, sum |s_out|} over this slab/batch. s_in and s_out must not alias. */
int nf_adjoint_prox(nf_plan* plan, const void* r_dev, const void* ymeas_dev, const void* s_in_dev,
                    void* s_out_dev, double eta_over_b, double alpha, double* stats_dev, void* stream);

/* Device flat sampler: idx[j] = pi_{seed,iter}(j) for j < batch, where pi is a keyed
 * Feistel bijection of [0, M). Distinct by construction; unordered.
 * iter == NF_ITER_DEVICE uses the plan's device-resident iteration counter and advances
 * it by one, so a captured CUDA graph of SPGM steps draws a fresh batch on every replay. */
#define NF_ITER_DEVICE 0xffffffffffffffffULL
int nf_sample_flat(nf_plan* plan, uint64_t seed, uint64_t iter, int batch, int32_t* idx_dev,
                   void* stream);

/* Structured sampler on the device: draws a Cartesian batch of n_f frequencies x n_tx
 * transmitters x n_rx receivers (distinct, sorted; keyed Feistel permutations of each axis, the
 * device counterpart of solver.sample_minibatch, solver.py:205-225, with its own RNG) and stages
 * it as nf_batch_prepare_structured would. iter = NF_ITER_DEVICE reads and advances the plan's
 * device iteration counter (capturable in a CUDA graph). lists (device, n_f + n_tx + n_rx), if
 * not null, receives the drawn [fs | ts | rs]. */
int nf_sample_structured(nf_plan* plan, uint64_t seed, uint64_t iter, int n_f, int n_tx, int n_rx,
                         int32_t* lists_dev, void* stream);

/* Persistent SPGM loop (the device-side loop of solver._solve, solver.py:259-318, for flat batches):
 * `iters` iterations in ONE cooperative launch (one CTA per SM, grid barriers between phases). Iteration k
 * draws its batch from idx_table[k*batch .. (k+1)*batch) (device int32, subset order, validated by the caller)
 * or, when idx_table is NULL, from the Feistel sampler with iteration number iter0 + k (nf_sample_flat), then
 * runs the same arithmetic as nf_batch_prepare + nf_forward + nf_adjoint_prox (bit-identical iterates).
 * Iteration k reads s_a (k even) or s_b (k odd) and writes the other buffer. records (device,
 * iters x 6 doubles) receives per iteration the nf_adjoint_prox statistics {sum|s|^2, sum(|s+|-|s|)^2,
 * D_B, sum|s+|} and the device time since launch [ns]. The loop stops early when
 * sqrt(stat1)/max(sqrt(stat0), 1e-12) < tol (solver.py:302, every CTA decides on the same bits) or when
 * time_budget_s >= 0 of device time has passed (checked after each iteration). state (device, 3 ints) =
 * {iterations run, reason: 0 all iterations / 1 tolerance / 2 time budget, budget flag}. Requirements:
 * batch <= max_batch, one forward window and batch <= 4096 (else NF_ERR_STATE; use the per-call path). */
int nf_spgm_loop(nf_plan* plan, const int32_t* idx_table_dev, int iters, uint64_t seed, uint64_t iter0, int batch,
                 const void* ymeas_dev, void* s_a_dev, void* s_b_dev, double eta_over_b, double alpha, double tol,
                 double time_budget_s, double* records_dev, int* state_dev, void* stream);

/* nf_spgm_loop for chained launches, so that a host can enqueue launch j + 1 before it reads launch j's state
 * (its Python solver draws and uploads the next chunk's batches and builds the last chunk's records while the GPU
 * runs): when prev_state_dev (device, the previous launch's state; NULL for the first) reports an early stop
 * (reason != 0), this launch runs no iteration and reports {0, that reason}; and every launch ends with the latest
 * iterate in s_a (an odd iteration count is copied back from s_b), so consecutive launches take the same
 * buffers. prev_state_dev and state_dev must differ. */
int nf_spgm_loop_chained(nf_plan* plan, const int32_t* idx_table_dev, int iters, uint64_t seed, uint64_t iter0,
                         int batch, const void* ymeas_dev, void* s_a_dev, void* s_b_dev, double eta_over_b,
                         double alpha, double tol, double time_budget_s, double* records_dev, int* state_dev,
                         const int* prev_state_dev, void* stream);

/* Set the plan's device iteration counter (stream-ordered). */
int nf_plan_set_iter(nf_plan* plan, uint64_t iter, void* stream);

/* Elementwise complex soft threshold over n values of the given dtype (v may alias out). */
int nf_soft_threshold(int dtype, const void* v_dev, void* out_dev, int64_t n, double alpha,
                      void* stream);

/* stats_dev (device, 2 doubles) = {sum |a|^2, sum (|b|-|a|)^2} over n values of the given
 * dtype, summed in a fixed order (deterministic). */
int nf_magnitude_change(int dtype, const void* a_dev, const void* b_dev, int64_t n,
                        double* stats_dev, void* stream);

/* Peer all-reduce of the forward partials over NVLink/NVSwitch (multi-GPU voxel-slab sharding,
 * SURVEY.md §8(e); the reference has no multi-GPU path, so nothing in it is replaced). One process per
 * GPU, one plan per rank over its z-slab:
 *   nf_comm_create        allocate this rank's receive slots and flags; write its CUDA IPC handle
 *                         (NF_IPC_HANDLE_BYTES bytes) to handle_out
 *   nf_comm_connect       map every peer's buffer; handles = world handles in rank order (the host
 *                         exchanges them, e.g. torch.distributed.all_gather_object)
 *   nf_forward_allreduce  nf_forward whose last reduce kernel pushes this rank's channel sums into every
 *                         rank's slots and sums all ranks' slots in rank order: y_dev is the FULL A_B s on
 *                         every rank (replaces nf_forward + an all-reduce of 2*B reals)
 *   nf_comm_status        *timed_out = 1 if a peer flag wait gave up (a rank stopped participating)
 *   nf_comm_emulate       test hook: `world` ranks emulated in one cooperative launch on the current GPU;
 *                         tmp_host [epochs][world][nseg][span][2] level-1 sums, y_host [epochs][world][span][2];
 *                         nseg = 0 runs the one-shot variant (structured batches): tmp_host [epochs][world][span][2]
 *                         is each rank's finished y */
#define NF_IPC_HANDLE_BYTES 64
int nf_comm_create(nf_plan* plan, int rank, int world, void* handle_out);
int nf_comm_connect(nf_plan* plan, const void* handles);
int nf_forward_allreduce(nf_plan* plan, const void* s_dev, void* y_dev, void* stream);
int nf_comm_status(nf_plan* plan, int* timed_out);
int nf_comm_emulate(int dtype, int world, int span, int nseg, int epochs, const double* tmp_host,
                    const int* sf_host, const int* spos_host, const double* pulse_host, int n_f, double* y_host);

const char* nf_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* NFGPU_H */
