/*
 * tpf.h — C ABI of the B200-native CommFuse hot path (libtpfuse_b200.so).
 *
 * This is the drop-in boundary for the reference's operator API
 * (/root/reference/proj/include/tpfuse/{collectives,layers}.hpp). Plain
 * pointers and sizes only; device pointers are raw CUDA device addresses,
 * streams are cudaStream_t passed as void*. All calls return 0 on success or a
 * negative TPF_E* code; the message is in tpf_last_error() (thread-local).
 *
 * Calls that move data are collective: every rank of a group must make the same
 * call (same shapes, schedule, granularity) in the same order on one stream.
 * There is no CPU fallback: without an sm_100 device every data-path call
 * fails with TPF_E_CUDA.
 */
#ifndef TPF_H_
#define TPF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes. The C++ mirror (include/tpfuse_b200/tpfuse.hpp) maps them to the
 * reference's exception types. */
#define TPF_OK 0
#define TPF_E_INVALID (-1)   /* std::invalid_argument (divisibility, granularity, peers)  */
#define TPF_E_SHAPE (-2)     /* tpfuse::ShapeError                                       */
#define TPF_E_LOGIC (-3)     /* std::logic_error (check_schedule)                         */
#define TPF_E_CUDA (-4)      /* CUDA runtime / launch failure, no device                  */
#define TPF_E_PEER (-5)      /* peer flag timeout: GroupError(rank, ...)                  */
#define TPF_E_CAPACITY (-6)  /* symmetric heap too small for this call                    */

/* ScheduleKind, collectives.hpp:19 */
#define TPF_RING 0
#define TPF_PAIRWISE 1
#define TPF_CIRCULAR 2

/* element types */
#define TPF_BF16 0
#define TPF_F32 1

/* AG-GEMM epilogue activation (tpsp_mlp_forward's element-wise Activation,
 * layers.hpp:58; only the exactly-representable ones run fused). */
#define TPF_ACT_NONE 0
#define TPF_ACT_SQUARE 1
/* Llama SwiGLU fused into the AG-GEMM epilogue: w is the tile-interleaved
 * gate||up shard — for every 256-column tile t, columns [256t, 256t+128) are
 * gate columns [128t, 128t+128) and [256t+128, 256t+256) the matching up
 * columns (N_local % 256 == 0). out is (B, S, N_local/2) = silu(gate) * up. */
#define TPF_ACT_SWIGLU 2

typedef struct tpf_comm tpf_comm;

int tpf_version(void);
const char* tpf_last_error(void);
/* number of SMs on the current device, 0 if no device */
int tpf_device_sms(void);

/* ---------------------------------------------------------- schedules (host)
 * Replaces: RingIndices ring_indices_ag/ring_indices_rs(int r, int i, int n)
 *           (collectives.hpp:51-55, collectives.cpp:47-55).
 * rs != 0 selects ring_indices_rs. out = {send_peer, recv_peer, compute_slice}. */
int tpf_ring_indices(int rs, int r, int i, int n, int32_t out[3]);

/* Replaces: Schedule build_schedule(ScheduleKind, int n)  (collectives.hpp:59,
 * collectives.cpp:57-107). out: n*n*3 int32, [rank][iteration](send, recv,
 * slice); nothing written for n == 1. Rejections as the reference:
 * TPF_E_INVALID for n < 1 or odd n with PAIRWISE. */
int tpf_schedule_build(int kind, int n, int32_t* out);

/* Replaces: void check_schedule(const Schedule&) (collectives.hpp:64,
 * collectives.cpp:180-235). TPF_E_LOGIC on a violated invariant. */
int tpf_schedule_check(int kind, int n, const int32_t* table);

/* -------------------------------------------------- communicator (RankEndpoint)
 * Replaces: RankEndpoint / RankGroup / spawn_group (fabric.hpp:114-226).
 * One process per GPU: each rank creates its communicator with a symmetric
 * heap of sym_bytes (device memory exported through CUDA IPC), exports its
 * handle, the caller exchanges the world's handles out of band (e.g. a
 * torch.distributed all_gather of the bytes), and opens them. */
#define TPF_IPC_HANDLE_BYTES 64
int tpf_comm_create(int rank, int world, size_t sym_bytes, tpf_comm** out);
int tpf_comm_ipc_handle(tpf_comm* c, void* handle_out /* TPF_IPC_HANDLE_BYTES */);
int tpf_comm_open_peers(tpf_comm* c, const void* handles /* world * TPF_IPC_HANDLE_BYTES */);

/* Single-GPU group: all `world` ranks are hosted by this process and every
 * fused call runs all ranks in ONE persistent launch (ranks own disjoint SM
 * sets; peer buffers are local). Used to prove the fused P2P protocol on one
 * GPU. Tensor arguments are then rank-stacked: x[world][...], w[world][...],
 * out[world][...]. */
int tpf_comm_create_local_group(int world, size_t sym_bytes_per_rank, tpf_comm** out);

/* Measurement tool: rank 0 of a `world`-rank group whose peers are virtual: their heaps
 * alias this rank's own heap (a self-ring), so each send fills the slot this rank reads one
 * step later and the ring's step-to-step waits are real from the first call, with zero link
 * latency. Runs the full per-rank protocol at full-GPU scale -- what one GPU of a TP group
 * computes. The results are well defined but are not a real group's: the AG gathers the own
 * slice at every step; the GEMM-RS sums the GEMMs of every row slice; the all-to-all
 * attention paths have no other sources and skip their receive waits. */
int tpf_comm_create_virtual(int world, size_t sym_bytes, tpf_comm** out);
/* Split group: `world` communicators on the current GPU, one per rank, each with its own
 * symmetric heap, device epoch and error record -- tpf_comm_create's per-process
 * communicator, with the other ranks' heaps mapped directly instead of through CUDA IPC.
 * Every fused GEMM call (tpf_ag_gemm, tpf_gemm_rs, tpf_dp_grad_rs, tpf_dp_param_ag_gemm) on
 * comms[r] builds rank r's launch exactly as the one-process-per-GPU path does (one hosted
 * rank, rank id r); the launch is deferred until every rank of the group has made the call,
 * and the last rank's call launches all of them as ONE grid (each rank on 148/world SMs), on
 * that call's stream. (Ranks whose kernels wait on each other must not be separate launches
 * on one GPU: nothing makes them co-resident.) Proves the per-rank protocol -- peer stores,
 * per-rank flags, epochs and waits -- on one GPU. Calls are collective in the reference's
 * sense (one worker per rank, fabric.hpp:185-226), issued here from one thread in rank order
 * or from any threads. comms: world pointers, destroyed one by one with tpf_comm_destroy. */
int tpf_comm_create_split_group(int world, size_t sym_bytes, tpf_comm** comms);
int tpf_comm_destroy(tpf_comm* c);
int tpf_comm_rank(const tpf_comm* c);
int tpf_comm_world(const tpf_comm* c);
/* CUDA device the communicator was created on (the library's current device at creation;
 * every call must run with that device current), -1 for a null handle */
int tpf_comm_device(const tpf_comm* c);
/* The rank that failed, as GroupError::failing_rank() (fabric.hpp:22-31): set by the last
 * tpf_comm_sync that returned TPF_E_PEER (-1 before). Waiters that give up record the rank
 * they were blocked on in every rank's blame table; sync follows that chain from the rank
 * that timed out to a rank that was not blocked (or that failed itself), so the victims of a
 * failure are not reported in its place. */
int tpf_comm_failing_rank(const tpf_comm* c);
/* Synchronise `stream` and check the device error record of every call since
 * the last check. TPF_E_PEER names the failing rank/step via tpf_last_error(). */
int tpf_comm_sync(tpf_comm* c, void* stream);
/* Test hook (fault injection, fabric_test.cpp:44-58 analogue): shrink the
 * peer-wait timeout (ns). 0 restores the default. */
int tpf_comm_set_timeout_ns(tpf_comm* c, int64_t ns);
/* Test hook: rank `rank` (-1 = none) stops publishing its peer flags, as if it
 * had failed mid-collective; its successors time out and tpf_comm_sync reports
 * TPF_E_PEER naming `rank` (tpf_comm_failing_rank). */
int tpf_comm_inject_fault(tpf_comm* c, int rank);
/* Measurement hook: on != 0 runs the same kernels over the same tile schedule with
 * every peer flag wait, wire store/load and ring forward disabled (results are
 * NOT the collective's). exposed comm = t(fused) - t(compute-only), SURVEY 8(d). */
int tpf_comm_set_compute_only(tpf_comm* c, int on);
/* Device timeline trace: buffer = device memory of (capacity+1) * 32
 * bytes, zeroed by the caller; word 0 counts records, record k (k >= 1) is
 * {kind | rank<<8 | block<<16 | step<<32, index, t0_ns, t1_ns} (%globaltimer).
 * Kinds: 1 tile epilogue, 2 producer main loop, 3 AG piece forwarded, 4 producer
 * wait on an AG wire image, 5 epilogue wait on an RS inbox, 6 RS flag published.
 * NULL disables (default). Used for the measured no-tail check. */
int tpf_comm_set_trace(tpf_comm* c, void* buffer, int64_t capacity_records);

/* -------------------------------------------------------------- fused ops
 * AG-GEMM. Replaces:
 *   Tensor column_parallel_forward(RankEndpoint&, const Tensor& x,
 *                                  const ShardedLinear& w, int m = 1)
 *       (layers.hpp:68-69, layers.cpp:120-127), i.e.
 *   Tensor fuse_all_gather(RankEndpoint&, const Tensor& x, f = matmul(., W_col[r]), m)
 *       (collectives.hpp:79-80, collectives.cpp:237-279).
 *   x   : bf16 (B, S/T, K) row-major — this rank's sequence slice
 *   w   : bf16 (K, N_local) row-major — this rank's column shard
 *   out : (B, S, N_local) row-major, out_dtype (TPF_BF16 | TPF_F32)
 * Ring schedule (ring_indices_ag), granularity m >= 1, S/T divisible by m. */
int tpf_ag_gemm(tpf_comm* c, const void* x, const void* w, void* out, int64_t B, int64_t S,
                int64_t K, int64_t N_local, int m, int act, int out_dtype, void* stream);

/* GEMM-RS. Replaces:
 *   Tensor row_parallel_forward(RankEndpoint&, const Tensor& x, const ShardedLinear& w,
 *                               const Schedule&, int m = 1)
 *       (layers.hpp:74-76, layers.cpp:129-138), i.e.
 *   Tensor fuse_reduce_scatter(RankEndpoint&, const Tensor& x, f = matmul(., W_row[r]),
 *                              const Schedule&, int m)  (collectives.hpp:87-89,
 *       collectives.cpp:362-405).
 *   x   : bf16 (B, S, K_local) row-major — this rank's feature shard
 *   w   : bf16 (K_local, N) row-major — this rank's row shard
 *   out : (B, S/T, N) row-major, out_dtype
 * kind: TPF_RING | TPF_PAIRWISE | TPF_CIRCULAR (reduction order exactly the
 * reference's); m > 1 only with TPF_RING; S divisible by T*m.
 * wire_dtype: dtype of the partial sums crossing NVLink (TPF_F32 for parity,
 * TPF_BF16 halves the bytes; rounds the running sum once per hop). */
int tpf_gemm_rs(tpf_comm* c, const void* x, const void* w, void* out, int64_t B, int64_t S,
                int64_t K_local, int64_t N, int kind, int m, int wire_dtype, int out_dtype,
                void* stream);

/* DP gradient sync (BASELINE cfg 4): reduce-scatter of the weight
 * gradient fused into its GEMM. Computes dW = sum_ranks X_r^T . dY_r (K x N) and
 * leaves rows [r*K/T, (r+1)*K/T) on rank r -- exactly
 *   fuse_reduce_scatter(x = X_r^T as (1, K, M_local), f = matmul(., dY_r), schedule, m)
 * (collectives.cpp:362-405), reduction order per schedule. X^T is read MN-major
 * straight from row-major X (no transpose).
 *   X  : bf16 (M_local, K) row-major     dY : bf16 (M_local, N) row-major
 *   dW : (K/T, N) row-major, out_dtype */
int tpf_dp_grad_rs(tpf_comm* c, const void* X, const void* dY, void* dW, int64_t M_local, int64_t K,
                   int64_t N, int kind, int m, int wire_dtype, int out_dtype, void* stream);

/* DP parameter all-gather fused into the forward GEMM (BASELINE cfg 4, a19): the
 * ring (ring_indices_ag) carries weight row blocks instead of activation chunks.
 * Rank r holds rows [r*N_local, (r+1)*N_local) of W (N x K, PyTorch Linear layout);
 * every rank computes its full output y = x . W^T, block l of the output columns in
 * ring step i with l = (r - i) mod T (fuse_all_gather order, collectives.cpp:237-279).
 *   x     : bf16 (M_local, K) row-major     w_rows : bf16 (N_local, K) row-major
 *   out   : (M_local, T*N_local) row-major, out_dtype */
int tpf_dp_param_ag_gemm(tpf_comm* c, const void* x, const void* w_rows, void* out, int64_t M_local,
                         int64_t K, int64_t N_local, int out_dtype, void* stream);
int64_t tpf_sym_bytes_dp_ag(int world, int64_t K, int64_t N_local);

/* UP / Ulysses attention with the output all-to-all fused (BASELINE cfg 5).
 * Replaces: Tensor fuse_all_to_all_attention(RankEndpoint&, const AttentionInputs&,
 *           const AttentionOptions&) (layers.hpp:100-101, layers.cpp:174-218).
 * Per rank (head group of `heads` heads, full sequence, Ulysses layout):
 *   q, k, v : bf16 (batch*heads, S, Dh)
 *   out     : bf16 (batch, S/T, T*heads*Dh) = concat_feat over source rank of merge_heads
 * Iteration i computes query slice l = (r+i+1) % T (softmax(q k^T * scale) v, scale =
 * 1/sqrt(Dh) if `scale`). Dh == 128 with (S/T) % 128 == 0 runs one fused tcgen05
 * flash-attention launch (S, P, O in TMEM) whose epilogue pushes every output tile straight
 * into rank l's buffer at this rank's feature block and flags it; other shapes run the GEMM
 * family (QK^T GEMM, softmax, P.V GEMM with the same push epilogue). The own slice is
 * computed last (no trailing transfer). Non-causal, no GQA. */
int tpf_attention_a2a(tpf_comm* c, const void* q, const void* k, const void* v, void* out, int64_t batch,
                      int64_t heads, int64_t S, int64_t Dh, int scale, void* stream);

// Ulysses first all-to-all (the ref_all_to_all step of
// layers_test.cpp:347-397, fabric.cpp:183-207): per rank q/k/v (batch*heads_total, S/T, Dh)
// bf16, sequence-sharded with every head -> q_out/k_out/v_out (batch*heads_total/T, S, Dh),
// this rank's head group over the whole sequence. Peer stores over NVLink + flags.
int tpf_ulysses_a2a(tpf_comm* c, const void* q, const void* k, const void* v, void* q_out, void* k_out, void* v_out,
                    int64_t batch, int64_t heads_total, int64_t S, int64_t Dh, void* stream);

// Whole UP layer (Ulysses attention, paper Alg. 5 with its first all-to-all): the first
// all-to-all above into the symmetric inbox, then fuse_all_to_all_attention (layers.cpp:174-218)
// reading straight from the inbox. q/k/v as tpf_ulysses_a2a; out (batch, S/T, heads_total*Dh)
// bf16. Needs Dh == 128 and (S/T) % 128 == 0.
int tpf_ulysses_attention(tpf_comm* c, const void* q, const void* k, const void* v, void* out, int64_t batch,
                          int64_t heads_total, int64_t S, int64_t Dh, int scale, void* stream);
// Symmetric heap bytes per rank that tpf_ulysses_attention, tpf_ulysses_a2a and
// tpf_attention_a2a (heads = heads_total / world) need; -1 on indivisible shapes.
int64_t tpf_sym_bytes_ulysses(int world, int64_t batch, int64_t heads_total, int64_t S, int64_t Dh);

/* Query-split attention (Alg. 4). Replaces:
 *   Tensor query_split_attention(RankEndpoint&, const AttentionInputs&, const ShardedLinear& out_proj,
 *                                const Schedule&, const AttentionOptions&)  (layers.hpp:88-91,
 *       layers.cpp:149-172)
 * = fuse_reduce_scatter over the query sequence of f(slice) = merge_heads(attention(q_slice, k, v)) . W_o[r].
 *   q, k, v : bf16 (batch*heads, S, 128)  this rank's head group, full sequence
 *   w_o     : bf16 (heads*128, D)         this rank's row shard of the output projection
 *   out     : (batch, S/T, D) out_dtype
 * The attention produces the context slice by slice in the RS schedule's order on part of the
 * SMs while, on a second stream, the fused GEMM-RS consumes each finished slice (per-slice
 * ready counters) on the rest: projection and transfer of step i run under the attention of
 * the later slices (Alg. 4). The reduction order is the schedule's. Graph-capturable. */
int tpf_query_split_attention(tpf_comm* c, const void* q, const void* k, const void* v, const void* w_o,
                              void* out, int64_t batch, int64_t heads, int64_t S, int64_t Dh, int64_t D, int kind,
                              int wire_dtype, int out_dtype, int scale, void* stream);

/* T == 1 degenerate case of both ops (collectives.cpp:242,379): out = a * b.
 *   a: bf16 (M, K), b: bf16 (K, N), out: (M, N) out_dtype. No communicator. */
int tpf_gemm(const void* a, const void* b, void* out, int64_t M, int64_t K, int64_t N,
             int out_dtype, void* stream);

/* Element-wise SwiGLU between the two fused ops of the Llama TP-SP MLP block
 * (tpsp_mlp_forward, layers.cpp:140-147, with the gate||up column shard):
 *   gu : bf16 (rows, 2*F) = [gate | up];  out: bf16 (rows, F) = silu(gate) * up */
int tpf_swiglu(const void* gu, void* out, int64_t rows, int64_t F, void* stream);

/* Bytes of symmetric heap a call needs (per rank), for sizing tpf_comm_create. */
int64_t tpf_sym_bytes_ag(int world, int64_t B, int64_t S, int64_t K, int64_t N_local, int m);
int64_t tpf_sym_bytes_rs(int world, int64_t B, int64_t S, int64_t K_local, int64_t N, int m,
                         int wire_dtype);

#ifdef __cplusplus
}
#endif
#endif /* TPF_H_ */
