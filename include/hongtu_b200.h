/*
 * hongtu_b200.h - C ABI of the B200-native HongTu GCN epoch path.
 *
 * The reference (`chunktrain`, /root/reference/pkg/src/chunktrain) is pure
 * Python/numpy and has no FFI of its own; every entry point below replaces
 * one Python-level operation of the reference and cites it (file:line,
 * relative to /root/reference/pkg/src/chunktrain/).  The Python package
 * `paper_2311_14898_b200` binds these with ctypes.
 *
 * Conventions
 *   - every function returns 0 on success, a negative HT_E* code on error;
 *     ht_last_error() returns the thread-local message of the last failure;
 *   - all buffers are plain pointers + int64 sizes; the caller owns every
 *     host array.  "Host" arrays passed to device operations must be pinned
 *     (ht_host_alloc or ht_host_register) or device-resident;
 *   - vertex ids, set members and index arrays are int64; edge weights are
 *     float64 on input (as the reference stores them, graph.py:141-150) and
 *     converted once to float32 for the device path;
 *   - integer preprocessing (graph build, LDG, chunks, plan sets, slots,
 *     reorganization) runs natively on the host CPU and is bit-exact with
 *     the reference.
 */
#ifndef HONGTU_B200_H
#define HONGTU_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HT_OK 0
#define HT_EINVAL (-1)     /* bad argument (maps to SimulationError/PlanError) */
#define HT_ECUDA (-2)      /* CUDA runtime failure                            */
#define HT_ESTATE (-3)     /* call out of sequence (SimulationError)         */
#define HT_ELIVE (-4)      /* row outside the live set (devices.py:177-187)   */
#define HT_ENOMEM (-5)

typedef struct ht_fleet ht_fleet; /* opaque: m virtual devices + uploaded plan */

/* ---- library / runtime -------------------------------------------------- */
const char* ht_last_error(void);
int ht_version(void);
int ht_device_count(int* count);

/* Pinned, portable, mapped host memory (HostStore backing, devices.py:47-57). */
int ht_host_alloc(int64_t bytes, void** out);
int ht_host_free(void* p);
int ht_host_register(void* p, int64_t bytes);
int ht_host_unregister(void* p);
/* Device-resident "host store" arrays for the HBM-resident (HongTu-IM) variant. */
int ht_dev_alloc(int device, int64_t bytes, void** out);
int ht_dev_free(int device, void* p);
int ht_memcpy(void* dst, const void* src, int64_t bytes); /* any direction, synchronous */
int ht_memset(void* dst, int value, int64_t bytes);

/* ---- integer preprocessing (host CPU, bit-exact) ----------------------- */

/* graph.py:91-150 from_edges + gcn_edge_weights: canonical CSC by
 * (dst, src), CSR by (src, dst), csr_edge_perm, float64 weights. */
int ht_build_graph(const int64_t* src, const int64_t* dst, int64_t E, int64_t V,
                   int64_t* csc_offsets, int64_t* csc_sources, int64_t* csr_offsets,
                   int64_t* csr_targets, int64_t* csr_edge_perm, double* weights);
/* Lean build for 10^9-edge synthetic graphs (synth_graph_streaming): int32
 * (src, dst) pairs, parallel edges removed (first of each (dst, src) pair,
 * synth.py:154-157), then the same canonical CSC / CSR / weights as
 * ht_build_graph.  Output edge arrays sized E; *e_out = edges kept. */
int ht_build_graph_dedup32(const int32_t* src, const int32_t* dst, int64_t E, int64_t V,
                           int64_t* csc_offsets, int64_t* csc_sources, int64_t* csr_offsets,
                           int64_t* csr_targets, int64_t* csr_edge_perm, double* weights,
                           int64_t* e_out);

/* CSR -> canonical edge permutation rebuilt from CSC + CSR offsets in one
 * counting pass (replaces the np.lexsort of graph.py:262-264 on HTG1 load). */
int ht_csr_perm(int64_t V, int64_t E, const int64_t* csc_offsets, const int64_t* csc_sources,
                const int64_t* csr_offsets, int64_t* perm);

/* synth.py:154-157 parallel-edge removal: indices (into src/dst) of the
 * first occurrence of each distinct (dst, src) pair, ascending by (dst, src),
 * i.e. np.unique(dst*V + src, return_index=True)[1].  keep holds E entries. */
int ht_dedup_edges(const int64_t* src, const int64_t* dst, int64_t E, int64_t V,
                   int64_t* keep, int64_t* n_keep);

/* partition.py:132-196 partition_vertices (LDG + one refinement sweep +
 * _repair_empty).  `arrival` is numpy default_rng(seed).permutation(V). */
int ht_ldg_partition(int64_t V, const int64_t* csc_offsets, const int64_t* csc_sources,
                     const int64_t* csr_offsets, const int64_t* csr_targets,
                     const int64_t* arrival, int64_t m, int64_t cap, int64_t* owner);

/* partition.py:235-267 chunk_from_vertices.  The caller sizes the edge
 * arrays with n_edges = sum of in-degrees of verts and `sources` with
 * n_edges entries (upper bound); *n_sources returns |N_ij|, and csr_off
 * must hold n_edges + 1 entries (only the first n_sources + 1 are used). */
int ht_chunk_fill(const int64_t* csc_offsets, const int64_t* csc_sources,
                  const double* weights, const int64_t* verts, int64_t nv,
                  int64_t* sources, int64_t* n_sources, int64_t* csc_off,
                  int64_t* csc_local_src, double* edge_w, int64_t* csr_off,
                  int64_t* csr_local_dst, int64_t* csr_perm);

/* Sorted-set algebra of planner.py:45-63 (inputs sorted unique int64).
 * op: 0 = intersect, 1 = difference (a \ b), 2 = union.  Returns the
 * output size through *n_out; out must hold |a|+|b| for union, |a| else. */
int ht_set_op(int op, const int64_t* a, int64_t na, const int64_t* b, int64_t nb,
              int64_t* out, int64_t* n_out);
int64_t ht_intersect_count(const int64_t* a, int64_t na, const int64_t* b, int64_t nb);

/* planner.py:252-284 build_buffer_layout for one device: given the n live
 * sets (sorted, concatenated with offsets), produce the slot of every live
 * row (aligned) and the capacity. */
int ht_slot_layout(int64_t n, const int64_t* live_concat, const int64_t* live_offsets,
                   int64_t* slots_concat, int64_t* capacity);

/* planner.py:386-450 reorganize (Alg. 4); nbr_concat/nbr_offsets hold the
 * m*n neighbour sets row-major [i][j].  Outputs chunk_orders (m*n, row-major
 * [i][pos]) and batch_order (n). */
int ht_reorganize(int64_t m, int64_t n, const int64_t* nbr_concat, const int64_t* nbr_offsets,
                  int move_all_rows, int64_t* chunk_orders, int64_t* batch_order);

/* ---- GPU dedup planner (K13): planner.py:292-315 build_plan on the device -
 * Input: the owner map (V) and, per chunk (i,j) row-major, the raw source
 * ids of its edges (duplicates allowed; src_offsets has m*n+1 entries).
 * Every set is computed on the GPU by radix sort / unique / membership and
 * is bit-identical with the host planner.  Sets come back concatenated in
 * this order (row-major over the indices named):
 *   N[i][j], U[j], T[i][j], carry[i][j], load[i][j], nbr_carry[i][j],
 *   fetch[i][j][k] (k != i, ascending; only when m > 1), live[i][j],
 *   slots[i][j] (aligned with live[i][j]);
 * caps has m entries (buffer capacities), volumes = (v_ori, v_p2p, v_ru). */
typedef struct ht_gplan ht_gplan;
int ht_gplan_build(int device, int m, int n, int64_t V, const int64_t* owner,
                   const int64_t* src_concat, const int64_t* src_offsets, ht_gplan** out);
int ht_gplan_count(ht_gplan* g, int64_t* nsets);
int ht_gplan_sizes(ht_gplan* g, int64_t* sizes, int64_t* caps, int64_t* volumes);
int ht_gplan_fetch(ht_gplan* g, int64_t* concat);
int ht_gplan_free(ht_gplan* g);

/* ---- fleet: m virtual devices executing one DedupPlan (devices.py) ----- */

#define HT_MODE_BASELINE 0
#define HT_MODE_P2P 1
#define HT_MODE_FULL 2
#define HT_FLUSH_ON_EVICTION 0
#define HT_FLUSH_EVERY_BATCH 1

/* DeviceFleet.__init__ (devices.py:132-171).  ordinals[i] = CUDA device of
 * virtual device i (several virtual devices may share one GPU). */
int ht_fleet_create(int m, int n, const int* ordinals, int mode, int flush_policy,
                    ht_fleet** out);
int ht_fleet_destroy(ht_fleet* f);

/* Rank mode (one process per GPU, torchrun): this process drives virtual
 * device `rank` on CUDA device `ordinal`; peers' slot buffers, gradient
 * views, weight-gradient accumulators and barrier counters are reached
 * through CUDA IPC, and the Alg. 2/3 barriers become device-side counter
 * waits (no host round trip).  Modes p2p/full only.  After the first
 * ht_epoch_begin, exchange HT_IPC_BYTES of handles with every peer. */
#define HT_IPC_BYTES 256
int ht_fleet_create_rank(int m, int n, int rank, int ordinal, int mode, int flush_policy,
                         ht_fleet** out);
int ht_fleet_ipc_export(ht_fleet* f, void* handles);
int ht_fleet_ipc_import(ht_fleet* f, int peer, const void* handles);

/* Plan sets of chunk (i, j) (planner.py:105-124).  live/slots aligned. */
int ht_fleet_set_sets(ht_fleet* f, int i, int j,
                      const int64_t* nbr, int64_t n_nbr,
                      const int64_t* owned, int64_t n_owned,
                      const int64_t* load, int64_t n_load,
                      const int64_t* nbr_carry, int64_t n_nbr_carry,
                      const int64_t* live, const int64_t* slots, int64_t n_live,
                      const int64_t* dest, int64_t n_dest /* -1: none */);
int ht_fleet_set_fetch(ht_fleet* f, int i, int j, int k, const int64_t* rows, int64_t n);
/* Chunk structure (partition.py:44-78) for the layer kernels. */
int ht_fleet_set_chunk(ht_fleet* f, int i, int j, int64_t nv, int64_t nn, int64_t ne,
                       const int64_t* csc_off, const int64_t* csc_local_src,
                       const double* edge_w, const int64_t* csr_off,
                       const int64_t* csr_local_dst, const int64_t* csr_perm);
/* Derive and upload every device index list (slot-translated CSC, copy
 * lists, push/flush lists).  Fails with HT_ELIVE if a set row is outside
 * its live set. */
int ht_fleet_finalize(ht_fleet* f);
int ht_fleet_capacity(ht_fleet* f, int i, int64_t* cap);

/* begin_forward_layer / begin_backward_layer (devices.py:193-207). */
int ht_begin_layer(ht_fleet* f, int dim, int elem_size, int backward);

/* dedup_comm_fwd (devices.py:223-278): stage batch rows (host loads,
 * barrier, staggered peer fetches, barrier) and copy each device's
 * N_ij view into views_out (concatenated over i). */
int ht_comm_fwd(ht_fleet* f, int batch, const void* host_rows, void* views_out);
/* dedup_comm_bwd (devices.py:284-341): push views (concatenated over i) to
 * owners in ascending source order, then flush per policy into host_grad. */
int ht_comm_bwd(ht_fleet* f, int batch, const void* views_in, void* host_grad);
/* load_dest_rows / store_dest_rows / add_dest_grads (devices.py:355-385):
 * op 0 load (host -> rows), 1 store (rows -> host), 2 add (host += rows). */
int ht_dest_rows(ht_fleet* f, int op, int batch, int dim, int elem_size,
                 void* host_rows, void* rows_concat);

/* ---- GCN epoch kernels (engine.py:387-480) ----------------------------- */

#define HT_PREC_FP32 0   /* SIMT FP32 GEMMs: FP32 validation mode (1e-5)      */
#define HT_PREC_TF32 1   /* tcgen05 TF32, 3xTF32 for z = agg.W (1e-3)         */

/* HBM owner cache: mode 0 off, 1 on (error if the
 * plan or free HBM does not allow it), 2 auto.  With it each device keeps
 * HBM mirrors of the host rows it owns (h^l, agg^l, grad_h^l) and the layer
 * calls read those instead of the host arrays; every produced row is still
 * written through to the host arrays.  Decided at each ht_epoch_begin;
 * ht_fleet_cache_state reports whether every local device uses it. */
int ht_fleet_set_cache(ht_fleet* f, int mode);
/* Compact host arrays (rank mode): the host arrays passed to the layer calls
 * hold only the local device's owned rows, ascending (`rows`, n = their
 * count; must equal the plan's owned rows); host row k = owned row k.  Needs
 * the HBM owner cache; host transfers become single contiguous copies.
 * rows == NULL restores full (V-row) host arrays. */
int ht_fleet_set_host_rows(ht_fleet* f, const int64_t* rows, int64_t n);
/* Lean epochs (opt-in): skip grad_h^0 (computed and
 * flushed by the reference, never consumed: engine.py:449, 477) and, with
 * the owner cache, the host copies of h^L and grad_h^L.  Weights, attention
 * vectors, loss and every other host array are unchanged. */
int ht_fleet_set_lean(ht_fleet* f, int lean);
/* Recompute-cache hybrid under an HBM budget (the paper's cache-vs-
 * recompute policy; the reference keeps every checkpoint,
 * devices.py:391-425): `bytes` caps what the owner cache may allocate per
 * device (0 = free HBM less 4 GB).  At each ht_epoch_begin the h^l and
 * grad_h^l mirrors must fit; agg^l mirrors are kept from the narrowest
 * layer up, and the layers that do not fit share one scratch buffer - their
 * agg^l is re-aggregated in the backward from the h^l mirror (the forward's
 * gather: bitwise the same rows, so epochs equal the all-cached ones).
 * Recompute needs one device with the identity mirror; otherwise the cache
 * is all or nothing.  ht_fleet_recompute_state: bit l set = agg^l recomputed
 * in the current epoch. */
int ht_fleet_set_budget(ht_fleet* f, int64_t bytes);
int ht_fleet_recompute_state(ht_fleet* f, int64_t* mask);
/* Checkpoint tier of the recompute-cache hybrid (replaces the host-side
 * cache of store_checkpoint / load_recomp_chkpt, devices.py:391-425): with
 * hbm = 1 and the owner cache active, a GCN forward keeps the agg
 * checkpoints in the HBM mirrors the backward reads and does not write them
 * to agg_out.  ht_fleet_checkpoint_read then fills host_agg (the layer's
 * (V, d_layer) host array) from the mirrors; valid until the next forward
 * of that layer.  With one device and one batch, TF32 layers with
 * d_out < d_in then run project-first (z = A.(h.W)); their agg^l is never
 * formed in the epoch and ht_fleet_checkpoint_read aggregates it on demand
 * (same kernel and edge order as the forward gather). */
int ht_fleet_set_checkpoints(ht_fleet* f, int hbm);
int ht_fleet_checkpoint_read(ht_fleet* f, int layer, void* host_agg);
/* HBM-resident store (HongTu-IM) on a single device: its device arrays
 * h[0..L], agg[0..L-1] (NULL for GAT), grad[0..L] are used as the owner
 * cache's mirrors (the layers read and write them in place, no copies).
 * h == NULL clears.  Takes effect at the next ht_(gat_)epoch_begin. */
int ht_fleet_alias_store(ht_fleet* f, int L, void* const* h, void* const* agg,
                         void* const* grad);
int ht_fleet_cache_state(ht_fleet* f, int* on);
/* Zero the per-device weight-gradient accumulators (engine.py:441-448). */
int ht_epoch_begin(ht_fleet* f, int L, const int* dims);
/* One forward layer over all batches (engine.py:409-434): dedup comm,
 * CSC aggregation, z = agg.W, ReLU, dest-row + checkpoint stores. */
int ht_forward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                     const void* h_in, void* h_out, void* agg_out, int precision);
/* downstream_loss (engine.py:297-320) on the last layer's device-resident
 * output; writes grad rows to grad_out (host.grad_h[L]).  count = mask.sum(). */
int ht_loss(ht_fleet* f, int d_last, const int64_t* labels, const uint8_t* mask,
            int64_t V, int64_t count, void* grad_out, double* loss);
/* Layer calls and ht_loss only enqueue work (no host synchronization);
 * with loss == NULL the value is read later with ht_loss_value, which
 * waits for the loss kernels. */
int ht_loss_value(ht_fleet* f, double* loss);
/* One backward layer over all batches (engine.py:449-477): checkpoint and
 * dest-gradient reload, hybrid backward, transposed aggregation, owner push
 * and flush into grad_in (host.grad_h[layer]). */
int ht_backward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                      const void* agg_in, const void* grad_out, void* grad_in,
                      int precision);
/* sync_and_update (engine.py:328-344): sum the device gradients in
 * ascending device order, W -= lr * sum (in place on the host arrays);
 * grads_out (may be NULL) receives the summed gradients. */
int ht_sgd(ht_fleet* f, int L, const int* dims, float* const* W, float lr,
           float* const* grads_out);
int ht_fleet_sync(ht_fleet* f);

/* ---- GAT epoch kernels (engine.py:196-289, 409-476; config 5) ---------- */
/* Replaces gat_layer_forward / gat_layer_backward_recompute and the GAT
 * branches of train_epoch (engine.py:418-423, 455-470) together with
 * DeviceFleet.load_dest_rows / add_dest_grads / load_recomp_chkpt("gat")
 * (devices.py:361-385, 427-432).  Widths must be multiples of 4 (<= 256
 * for HT_PREC_TF32).  A = attention vector [a_dst | a_src] (2 d_out). */
int ht_gat_epoch_begin(ht_fleet* f, int L, const int* dims);
/* One forward layer over all batches: dedup comm of h_in rows, destination
 * input rows, q = h_nbr.W / p = h_dst.W (3xTF32), edge softmax
 * aggregation, ReLU, destination rows stored to h_out (host.h[l+1]). */
int ht_gat_forward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                         const float* A, float slope, const void* h_in, void* h_out,
                         int precision);
/* One recompute-backward layer over all batches: inputs re-staged through
 * the forward machinery, destination inputs and gradients loaded, layer
 * recomputed and differentiated; destination-input gradients added into
 * grad_in (host.grad_h[l]), neighbour gradients pushed to owners and
 * flushed (read-modify-write: grad_in must be zero at epoch start). */
int ht_gat_backward_layer(ht_fleet* f, int layer, int d_in, int d_out, const float* W,
                          const float* A, float slope, const void* h_in,
                          const void* grad_out, void* grad_in, int precision);
/* ht_sgd plus the attention vectors (engine.py:339-343); A, gW_out, gA_out
 * may be NULL. */
int ht_sgd2(ht_fleet* f, int L, const int* dims, float* const* W, float* const* A, float lr,
            float* const* gW_out, float* const* gA_out);

/* ---- timing of the dominant kernels (bench roofline) ------------------- */
/* Enables CUDA-event timing of the aggregation kernels; ht_kernel_stats
 * returns launches, summed milliseconds and summed algorithmic bytes of
 * kernel class `which` (0 = forward CSC aggregation, 1 = backward CSR
 * aggregation, 2 = GEMMs, 3 = host transfers) since the last reset. */
int ht_set_timing(ht_fleet* f, int enabled);
int ht_kernel_stats(ht_fleet* f, int which, int64_t* launches, double* ms, double* bytes);

/* Device-timeline marks: record event `which` (0 = start, 1 = stop) on
 * every device stream; ht_fleet_elapsed returns the max over devices of
 * stop - start in milliseconds (bench.py's CUDA-event timing). */
int ht_fleet_mark(ht_fleet* f, int which);
int ht_fleet_elapsed(ht_fleet* f, double* ms);
/* Marks 0..15 may be recorded; elapsed time from mark a to mark b (max over
 * devices) - per-phase device timing. */
int ht_fleet_elapsed_between(ht_fleet* f, int a, int b, double* ms);
/* Number of kernels this library has launched (process-wide). */
int64_t ht_launches(void);

/* PCIe peaks of the box in GB/s (roofline denominators of the transfer
 * kernels): out[0] copy-engine H2D, out[1] D2H, out[2] both directions at
 * once (sum), out[3] zero-copy row kernel reading pinned memory, out[4]
 * zero-copy row kernel writing pinned memory.  `bytes` per transfer. */
int ht_pcie_probe(int device, int64_t bytes, double* out);

/* GEMM unit entry for tests: runs the launchers the layer drivers use on
 * host arrays (device 0).  op 0: C = relu(A W); 1: C = [A W > 0] * G;
 * 2: C = A W^T (A: M x N, W: K x N); 3: C = A^T G (A: M x K, G: M x N);
 * 4: C = (G * [A > 0]) W^T, 5: C = the TF32-rounded G * [A > 0] that op 4
 * writes beside it (A: M x N; TF32 only - the backward's ReLU'-masked GEMM).
 * precision HT_PREC_FP32 (SIMT) or HT_PREC_TF32 (tcgen05). */
int ht_gemm_test(int op, int precision, const float* A, const float* W, const float* G,
                 float* C, int64_t M, int K, int N);

/* GEMM rate (measurement, no reference counterpart): `iters` back-to-back
 * launches of the layer drivers' GEMM launcher `op` (0, 2, 3 as above) on
 * device-resident M-row operands.  out[0] ms per launch, out[1] TFLOP/s of
 * the useful 2*M*K*N flops, out[2] GB/s of the operand rows read once. */
int ht_gemm_rate(int op, int precision, int64_t M, int K, int N, int iters, double* out);

/* Profiler range (measurement): start != 0 -> cudaProfilerStart, else
 * cudaProfilerStop.  bench.py --profile-epoch brackets one epoch with it so
 * `ncu --replay-mode app-range --profile-from-start off` reads the PCIe /
 * NVLink / DRAM counters of exactly that epoch (kernels and copy engines). */
int ht_profile_range(int start);

/* Free and total HBM of `device` in bytes (cudaMemGetInfo): sizing an
 * hbm_budget for DeviceFleet, bench diagnostics. */
int ht_mem_info(int device, int64_t* free_bytes, int64_t* total_bytes);

#ifdef __cplusplus
}
#endif
#endif
