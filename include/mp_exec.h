/*
 * mp_exec.h — C-ABI of the B200 plan executor (libmpexec.so).
 *
 * The reference (meshplan, pure Python) has no native boundary: its executor is
 * the discrete-event simulator `simulate` (reference pkg/src/meshplan/sim.py:91-188),
 * which advances a clock by a modeled `duration` for every `compute` instruction
 * (reshard.py:382, sim.py:148-151) and by `transfer_time`/`collective_time` for
 * every `send`/`all_gather` (sim.py:74-88).  The functions below are the device
 * work those instructions stand for.  Each entry point cites the reference site
 * whose modeled cost it replaces with real sm_100a work.
 *
 * Conventions
 *   - plain pointers / sizes only; no torch types;
 *   - every call takes a `void* stream` (a cudaStream_t; NULL = legacy stream);
 *   - return 0 on success, non-zero on error; `mp_last_error()` returns the
 *     per-thread message of the last failure;
 *   - tensors are row-major with explicit element strides; bf16 = uint16 bits.
 *
 * Binding from the reference side is via ctypes (the reference is Python);
 * see INTEGRATION.md.
 */
#ifndef MP_EXEC_H
#define MP_EXEC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ------------------------------------------------------------ */

/* ABI version (bumped on signature changes). */
int mp_abi_version(void);

/* Message of the last failed call on this thread ("" if none). */
const char* mp_last_error(void);

/* Number of device kernels this library has launched since load (all entry
 * points; used by bench.py for the `gpu_launches` claim). */
uint64_t mp_launch_count(void);
/* Load every libmpexec kernel now (CUDA lazy module loading would load a kernel at
 * its first launch, blocking the host while an NCCL kernel spins on the device).
 * Called once per process by the executor; 0 ok. */
int mp_preload_kernels(void);

/* ---- GEMM ------------------------------------------------------------------
 * Replaces the modeled local matmul of a chosen ParallelAlgorithm
 * (sharding.py:255-299; its time is compute_time, costs.py:83-86) and the
 * batched variant (loops b,i,j,k, sharding.py:217-218).
 *
 *   C[b0,b1] = alpha * A[b0,b1] @ B[b0,b1] + beta * C[b0,b1]      (fp32 accumulate)
 *
 * Operand descriptors are int64[6]:
 *   {rows, cols, row_stride, col_stride, batch_stride0, batch_stride1}
 * in elements, describing the LOGICAL operand (A is M x K, B is K x N, C is M x N).
 * For A and B exactly one of row_stride / col_stride must be 1 (K-major or
 * MN-major storage; both are read by TMA with 128-byte swizzle straight into
 * the tcgen05 operand layout, so transposed operands are never materialised).
 * C must have col_stride == 1.  A, B: bf16.  C: bf16 (c_dtype 0) or fp32 (1).
 * epilogue: 0 none, 1 GeLU(tanh) applied to alpha*acc (beta must be 0).
 */
int mp_gemm_bf16(const void* A, const int64_t* a_desc,
                 const void* B, const int64_t* b_desc,
                 void* C, const int64_t* c_desc, int c_dtype,
                 int64_t nbatch0, int64_t nbatch1,
                 float alpha, float beta, int epilogue,
                 void* stream);
/* Same with fused epilogues on an auxiliary bf16 matrix (same M x N extents
 * and batch structure as C; aux_desc = {row_stride, batch_stride0,
 * batch_stride1}).  beta must be 0.
 *   2: C = alpha*acc + aux            residual add / gradient accumulation
 *                                     (the add member, graph.py:305,311,328-332)
 *   3: C = alpha*acc * gelu'(aux)     GeLU backward on the dX of the next matmul
 *   4: C = alpha*acc; aux <- gelu(C)  pre-activation and activation in one pass */
int mp_gemm_bf16_ex(const void* A, const int64_t* a_desc,
                    const void* B, const int64_t* b_desc,
                    void* C, const int64_t* c_desc, int c_dtype,
                    int64_t nbatch0, int64_t nbatch1,
                    float alpha, float beta, int epilogue,
                    void* aux, const int64_t* aux_desc, void* stream);

/* ---- elementwise / row ops (trivial members, intra.py:93-160) ------------- */

/* y = gelu_tanh(x); bf16, n elements, contiguous. */
int mp_gelu_fwd(const void* x, void* y, int64_t n, void* stream);
/* dx = gelu_tanh'(x) * dy; bf16. */
int mp_gelu_bwd(const void* x, const void* dy, void* dx, int64_t n, void* stream);
/* y = a + b (bf16, contiguous). */
int mp_add(const void* a, const void* b, void* y, int64_t n, void* stream);
/* y = scale * x (bf16 -> bf16), used for the loss seed dL/dy. */
int mp_scale(const void* x, void* y, float scale, int64_t n, void* stream);
/* Sum of squares of x (bf16) accumulated into out[0] (fp32, atomically). */
int mp_sumsq(const void* x, float* out, int64_t n, void* stream);

/* Row softmax over the last dim of a [rows, cols] bf16 matrix (row stride ld),
 * y = softmax(scale * x).  Complete rows only (softmax dim not split). */
int mp_softmax_fwd(const void* x, void* y, int64_t rows, int64_t cols, int64_t ld,
                   float scale, void* stream);
/* Split-row variant (softmax dim sharded over a mesh axis, SURVEY §7 hard
 * part 3).  stats: fp32 planar [3, rows] = (row max, row sum-exp, max copy).
 *   mp_softmax_stats   local partials of the local columns
 *   (caller: MAX all-reduce of stats[0:rows])
 *   mp_softmax_rescale sum *= exp(local max - group max)
 *   (caller: SUM all-reduce of stats[rows:2*rows])
 *   mp_softmax_apply   y = exp(scale*x - max) / sum */
int mp_softmax_stats(const void* x, float* stats, int64_t rows, int64_t cols,
                     int64_t ld, float scale, void* stream);
int mp_softmax_rescale(float* stats, int64_t rows, void* stream);
int mp_softmax_apply(const void* x, const float* stats, void* y, int64_t rows,
                     int64_t cols, int64_t ld, float scale, void* stream);
/* dx = scale * y * (dy - rowsum(dy*y)); rowdot: optional fp32 [rows] holding
 * the (already all-reduced) rowsum, or NULL to compute it locally. */
int mp_softmax_bwd(const void* y, const void* dy, void* dx, const float* rowdot,
                   int64_t rows, int64_t cols, int64_t ld, float scale, void* stream);
/* rowdot[r] = sum_c dy[r,c]*y[r,c]  (fp32 out), for the split-row backward. */
int mp_softmax_rowdot(const void* y, const void* dy, float* rowdot, int64_t rows,
                      int64_t cols, int64_t ld, void* stream);

/* ---- fused attention (cluster bmm -> softmax -> bmm, graph.py:297-302, and its
 * structural backward graph.py:341-361), for stages whose softmax dim is local.
 * Q/K/V/O/dO/dK/dV: (B*s, ld) bf16 row-major, head hh in columns [hh*d, hh*d+d);
 * d must be 64, s a multiple of 128.  lse, dvec: fp32 [B*H, s].  dq_acc: fp32
 * (B*s, ld), zeroed by the call itself (its D pre-pass), then accumulated by TMA bulk
 * reductions (cast afterwards).
 * Non-causal softmax(scale * q k^T). */
int mp_attn_fwd(const void* q, const void* k, const void* v, void* o, float* lse,
                int64_t B, int64_t H, int64_t s, int64_t d, int64_t ld, float scale,
                void* stream);
int mp_attn_bwd(const void* q, const void* k, const void* v, const void* o,
                const void* dout, const float* lse, float* dvec, float* dq_acc,
                void* dk, void* dv, int64_t B, int64_t H, int64_t s, int64_t d,
                int64_t ld, float scale, void* stream);

/* Key-range variants for stages that shard the softmax (key) dim of the
 * scores over a mesh axis (spec RRS^a on the cluster's bmm/softmax nodes):
 * only keys [kv0, kv0+kv_len) of every sequence are read (128-aligned).  fwd
 * writes O / LSE normalised over that range; bwd writes dK / dV rows of the
 * range and accumulates dq_acc over it, given the GLOBAL lse (and full O, dO). */
int mp_attn_fwd_kv(const void* q, const void* k, const void* v, void* o, float* lse,
                   int64_t B, int64_t H, int64_t s, int64_t d, int64_t ld, float scale,
                   int64_t kv0, int64_t kv_len, void* stream);
int mp_attn_bwd_kv(const void* q, const void* k, const void* v, const void* o,
                   const void* dout, const float* lse, float* dvec, float* dq_acc,
                   void* dk, void* dv, int64_t B, int64_t H, int64_t s, int64_t d,
                   int64_t ld, float scale, int64_t kv0, int64_t kv_len, void* stream);
/* Combine of key-split partial attention (between the collectives over the key
 * axis): scale: w = exp(lse - m), o *= w (m = max-allreduced lse);
 * finish: o /= wsum, lse = m + log(wsum) (wsum = sum-allreduced w). */
int mp_attn_combine_scale(void* o, const float* lse, const float* m, float* w, int64_t B,
                          int64_t H, int64_t s, int64_t d, int64_t ld, void* stream);
int mp_attn_combine_finish(void* o, const float* wsum, const float* m, float* lse,
                           int64_t B, int64_t H, int64_t s, int64_t d, int64_t ld,
                           void* stream);

/* ---- GShard top-2 routing (MoE builder, paper_2201_12023_b200/builders.py) ---
 * The MoE graph's gates -> (G, E*C, S) dispatch-mask and gates -> (G, S, E*C)
 * combine-weight reshapes (graph.py:240-245 layout adapters; the reference has
 * no MoE builder).  route: int32 [tokens, 4] = {e1, pos1|-1, e2,
 * pos2|-1} per token, groups of S tokens, capacity C (rule in csrc/moe.cu).
 * mask mode 0: dispatch ones, mode 1: combine gate weights; `out` is fully
 * written.  mask_grad (T, E) bf16: mode 1 out[t, e] = d at the routed slot of
 * (t, e), else 0; mode 0 zeros (the 0/1 dispatch mask has no gradient). */
int mp_moe_route(const void* gates, int64_t ld, int64_t groups, int S, int E, int C,
                 int* route, void* stream);
int mp_moe_mask(const int* route, const void* gates, int64_t ld, void* out, int64_t tokens,
                int S, int E, int C, int mode, void* stream);
int mp_moe_mask_grad(const int* route, const void* d, void* out, int64_t tokens, int S, int E,
                     int C, int mode, void* stream);

/* ---- Wide-ResNet layout adapters (builders.build_wide_resnet; the IR has no
 * convolution): NHWC activations (rows (n, y, x), columns c), bf16.
 * im2col: k x k (odd) window, stride s, zero padding k/2 -> rows (n, oy, ox),
 * columns (ky, kx, c); backward=1 is its adjoint col2im (x = d columns,
 * out = (N*H*W, C)).  subsample: out = in at (oy*s, ox*s); backward scatters into
 * zeros.  reduce_mid: (A, B, C) -> (A, C) sum over B (the head's pooling
 * reduction, graph.py:232-237); broadcast=1 its backward (A, C) -> (A, B, C). */
int mp_im2col(const void* x, void* out, int64_t N, int64_t H, int64_t W, int64_t C, int k,
              int s, int backward, void* stream);
int mp_subsample(const void* x, void* out, int64_t N, int64_t H, int64_t W, int64_t C, int s,
                 int backward, void* stream);
int mp_reduce_mid(const void* x, void* out, int64_t A, int64_t B, int64_t C, int broadcast,
                  void* stream);

/* ---- box pack / unpack (cross-mesh Transfer, reshard.py:32-37,97-108) -----
 * Copies the sub-box [lo, lo+ext) of a strided tensor of rank <= 4 to / from
 * a dense buffer.  dims/strides in elements, elem_bytes in {2,4}. */
int mp_pack_box(const void* src, const int64_t* src_strides, const int64_t* lo,
                const int64_t* ext, int rank, int elem_bytes, void* dst, void* stream);
int mp_unpack_box(const void* src, void* dst, const int64_t* dst_strides,
                  const int64_t* lo, const int64_t* ext, int rank, int elem_bytes,
                  void* stream);

/* ---- NCCL communicators (owned by the library, driven on the caller's stream,
 * capturable in CUDA graphs).  Replace the modeled collective_time /
 * transfer_time of the reference (costs.py:63-92).  dtype: 0 bf16, 1 fp32,
 * 2 bytes.  op: 0 sum, 1 max.  Peers are ranks within the communicator. */
int mp_nccl_version(void);
int mp_nccl_unique_id(void* out128);
int mp_comm_init(const void* uid128, int nranks, int rank, void** comm_out);
int mp_comm_destroy(void* comm);
/* Release a hung communicator (every pending operation on it fails) and poll a
 * communicator's asynchronous error state without blocking; nccl_result gets the
 * ncclResult_t (0 ok).  The executor's watchdog uses them to turn a hang into an
 * ExecError naming the blocked instruction (the deadlock SimError of
 * sim.py:172-178). */
int mp_comm_abort(void* comm);
int mp_comm_async_error(void* comm, int* nccl_result);
int mp_allreduce(void* comm, void* buf, int64_t count, int dtype, int op, void* stream);
int mp_allgather(void* comm, const void* send, void* recv, int64_t sendcount, int dtype,
                 void* stream);
/* ZeRO realisation of a gradient all-reduce (intra.py:404-424 post_ilp_rewrite):
 * reduce-scatter of `recvcount * nranks` elements, rank r keeps chunk r. */
int mp_reduce_scatter(void* comm, const void* send, void* recv, int64_t recvcount, int dtype,
                      int op, void* stream);
int mp_group_start(void);
int mp_group_end(void);
/* All-to-all of equal chunks: chunk i (count elements) of send goes to rank i, chunk i of
 * recv comes from rank i (one NCCL group of sends and recvs).  Replaces the modeled
 * all_to_all of resharding_cost (sharding.py:346; collective_time, costs.py:63-73). */
int mp_alltoall(void* comm, const void* send, void* recv, int64_t count, int dtype, void* stream);
int mp_send(void* comm, const void* buf, int64_t count, int dtype, int peer, void* stream);
int mp_recv(void* comm, void* buf, int64_t count, int dtype, int peer, void* stream);

/* ---- optimizer (weight update after the ZeRO rewrite, intra.py:404-424) ---
 * Fused Adam over flat fp32 master/m/v/grad buffers, writing the bf16
 * working copy; grad is scaled by grad_scale before use. */
int mp_adam_step(float* master, float* m, float* v, const float* grad,
                 void* param_bf16, int64_t n, float lr, float beta1, float beta2,
                 float eps, float weight_decay, float grad_scale, int64_t step,
                 void* stream);

/* fp32 -> bf16 and bf16 -> fp32 casts (n elements, contiguous). */
int mp_cast_f32_bf16(const float* x, void* y, int64_t n, void* stream);
int mp_cast_bf16_f32(const void* x, float* y, int64_t n, void* stream);
/* y(fp32) += x(bf16)  (gradient accumulation of a bf16 partial). */
int mp_accum_bf16_f32(const void* x, float* y, int64_t n, void* stream);
/* Split-K reduction for gradient GEMMs with few output tiles (e.g. the MoE
 * 1024x1024 attention dW): y = beta*y + sum_p parts[p*n : (p+1)*n], in order. */
int mp_sum_parts_f32(const float* parts, int64_t nparts, int64_t n, float* y, float beta,
                     void* stream);

/* ---- planner acceleration --------------------------------
 * Exact branch-and-bound of the intra-op strategy ILP with the reference's
 * semantics (intra.py:323-401: greedy incumbent, suffix bound, index-order DFS,
 * strict improvement, node budget).  Host-only (no device work).  Costs are
 * integers in one common unit (the caller scales the exact rationals). */
int mp_ilp_solve(int n, const int* k, const int64_t* costs, int n_edges, const int* u,
                 const int* v, const int64_t* mats, int64_t budget, int* choice_out,
                 int64_t* objective_out, int* certified_out, int64_t* explored_out);

#ifdef __cplusplus
}
#endif
#endif /* MP_EXEC_H */
