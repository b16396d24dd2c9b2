/*
 * rrs.h — C-ABI of the B200-native Rotated Runtime Smooth (RRS) A4W4 linear layer.
 *
 * Method: "Rotated Runtime Smooth: Training-Free Activation Smoother for accurate INT4 inference"
 * (arXiv 2409.20361).  Citations are PAPER.md line numbers (P:n) with section/equation, and the
 * readings R1..R24 of DESIGN.md §3 where the paper is silent.
 *
 * Notation: T tokens (paper's N), K input features, N output features (paper's M),
 * group size L = 128 (= GEMM K-block; any power of two in [32, 1024] is accepted, the
 * group sizes of the paper's Table 4 ablation), G = K / L groups.
 *
 * Conventions shared by every entry point
 *   - Array arguments are DEVICE pointers (CUDA global memory) allocated and owned by the caller;
 *     the library never allocates on the hot path and never frees caller memory.  Scratch comes
 *     from a caller-provided workspace `ws` of at least rrs_workspace_bytes(...) bytes.
 *   - Row-major, innermost dimension contiguous: X[T][K], W[N][K] (nn.Linear layout), Y[T][ldy].
 *   - bf16 / f32 data is passed as raw bits (uint16_t for bf16); dtype enums select the format.
 *   - Packed INT4 (D4): uint8 [rows][K/2]; byte b holds code 2b in bits 0..3 and code 2b+1 in bits
 *     4..7, two's-complement nibbles; codes lie in [-7, 7] (clamp [-8, 7], R11).
 *   - GEMM operand layout ("Xop"/"Wop"): uint8 [rows][K], one code per byte, columns in the REORDERED
 *     order j'.  sm_100a has no INT4 MMA, so each code is widened to one byte (DESIGN.md §6/§7):
 *       default          the byte is the E4M3 encoding of the code (exact: |q| <= 8), consumed by
 *                        tcgen05 .kind::f8f6f4 whose FP32 group sums are exact integers (|P_g| < 2^13);
 *       RRS_OPERAND_I8   the byte is the int8 code, consumed by tcgen05 .kind::i8 (int32 sums).
 *     Producer (rrs_prepare_weights / rrs_rotate_smooth_quant) and consumer (rrs_gemm / rrs_linear)
 *     must be called with the same RRS_OPERAND_I8 flag.
 *   - Every call enqueues work on `stream` (a cudaStream_t, NULL = legacy default stream) and
 *     returns without synchronising the host.  Asynchronous device faults surface on a later CUDA call.
 *   - Validation happens before any launch; on error nothing is enqueued, the status is returned
 *     and rrs_last_error() (thread-local) describes it.
 *   - Supported shapes: group a power of two in [32, 1024] dividing K; K % 128 == 0 and K in {128,256,...,16384} (2^m) or
 *     {7168, 14336} (28*2^m, R2); T >= 0; N >= 1.  All pointers 16-byte aligned.
 *   - X must be bf16 and satisfy the exactness precondition of DESIGN.md R3 (per row, exponent span
 *     of the nonzero |x| <= 45 - ceil(log2 K)); NaN/Inf inputs are undefined behaviour (not checked).
 *   - Reentrant.  Library state: per-device caches (device properties, occupancy, kernel attributes) behind a
 *     mutex; the decode prologue's grid-barrier counters (256 slots in device memory, zero at load, reset by every
 *     use, one slot per call from an atomic counter -- a CUDA graph captures its slot, so concurrent replays of ONE
 *     graph on several streams are not supported); the NCCL communicator objects the caller creates.
 */
#ifndef RRS_H_
#define RRS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RRS_OK = 0,
  RRS_ERR_INVALID_ARGUMENT = 1,  /* null pointer where required, negative size, group not a power of two
                                    in [32, 1024] */
  RRS_ERR_UNSUPPORTED_SHAPE = 2, /* K not 2^m / 28*2^m, K % group != 0 or K % 128 != 0 (R7) */
  RRS_ERR_MISALIGNED = 3,        /* pointer or leading dimension not 16-byte aligned */
  RRS_ERR_WORKSPACE_TOO_SMALL = 4,
  RRS_ERR_ARCH = 5,              /* current device is not sm_100 (B200) */
  RRS_ERR_CUDA = 6,              /* a CUDA runtime/driver call failed (message in rrs_last_error) */
  RRS_ERR_NCCL = 7               /* an NCCL call failed */
} rrs_status;

typedef enum { RRS_BF16 = 0, RRS_F32 = 1 } rrs_dtype;

/* flags */
#define RRS_GEMM_PLAIN 0x1u   /* rrs_gemm: per-channel A4W4 baseline: one sum over all K, no s_g */
#define RRS_OPERAND_I8 0x2u   /* GEMM operands are int8 codes (tcgen05 .kind::i8) instead of E4M3 bytes */
#define RRS_GEMM_SWIGLU 0x8u  /* rrs_gemm / rrs_linear: fused SwiGLU epilogue, see rrs_gemm */
#define RRS_GEMM_SUBCHANNEL 0x10u /* rrs_gemm: sub-channel A4W4 baseline, see rrs_gemm */
#define RRS_TOKEN_SHARDED 0x4u /* rrs_linear with comm: token-sharded data parallel, see below */
#define RRS_NO_ROTATION 0x40u /* plain Runtime Smooth (Eq. 1-3): no Hadamard on X (prologue) nor
                                 on W (rrs_prepare_weights); rrs_linear then uses out_scale 1 */
#define RRS_PREROTATED 0x80u  /* X arrives already rotated (QuaRot-style rotation fused upstream): the prologue
                                 skips a1; W is prepared as usual (rotated); rrs_linear keeps out_scale 1/K */
#define RRS_NO_SMOOTH 0x100u  /* efficiency baselines only (SURVEY §8(d) O_quarot / O_plain): skip a2-a5, s_g = 1,
                                 i.e. per-token RTN of X~ (with RRS_NO_ROTATION: of X) */
#define RRS_W_PACKED4 0x20u   /* decode regime (configs[3], T <= 64): W kept PACKED at 4 bits ("decode4" layout), see
                                 rrs_prepare_weights / rrs_gemm / rrs_linear */

typedef struct rrs_comm_s* rrs_comm_t;

/* Human-readable status name; never NULL. */
const char* rrs_status_str(int status);
/* Detail of the last error raised on the calling thread ("" if none). */
const char* rrs_last_error(void);
/* ABI version (major * 100 + minor); 101 added RRS_W_PACKED4, 102 RRS_NO_ROTATION / RRS_PREROTATED / RRS_NO_SMOOTH. */
int rrs_version(void);

/* Workspace bytes needed by rrs_linear / rrs_rotate_smooth_quant for T tokens:
 * X~[T][K] f32 (the rotated activation, written once by the FWHT pass and read by the quantisation
 * pass) + chan_max[K] f32 + s_group[G] f32 + x_scale[T] f32 + Xop[T][K] u8 (+ split-K partials
 * 8 * T * N f32 for decode-sized T <= 128 without a communicator when N % 4 == 0 and N <= 19200, the shapes whose
 * single-GPU GEMM may split K; + Y shard and gather buffers when world > 1), each 256-byte aligned.  Returns 0 for
 * invalid arguments. */
size_t rrs_workspace_bytes(int64_t T, int64_t N, int64_t K, int32_t group, int32_t world);
/* Workspace for rrs_linear / rrs_allgather_columns WITH a communicator of `world` ranks (world >= 1; a 1-rank
 * communicator still runs the NCCL path): as above plus the Y shard and all-gather buffers, always. */
size_t rrs_workspace_bytes_comm(int64_t T, int64_t N, int64_t K, int32_t group, int32_t world);

/* Offline reorder helper ("reorder the activations and weights according to the magnitude
 * of smoothing scales"; R5, R21): perm[j'] = channel of rank j' when channels are sorted by
 * chan_max descending, ties by ascending channel index.  chan_max: device f32 [K] (>= 0),
 * typically the rotated calibration activation's chan_max output; perm: device int32 [K]. */
rrs_status rrs_perm_from_channel_max(const float* chan_max, int64_t K, int32_t* perm, void* stream);

/* Offline weight preparation ("offline rotate the weight matrix", weights
 * quantised per output channel with symmetric RTN, R12/R13; P:109 step 1 reorders W like X):
 *   W~ = W . H_K (exact, R1-R3) -> columns permuted by perm (never scaled)
 *   beta_n = fl(max_j |W~_nj| / 7) (1 if the row is zero, R8); codes rint_even(fl(W~ * fl(7/max))).
 * W: device bf16 bits [N][K].  perm: device int32 [K] (NULL = identity is NOT accepted: pass it).
 * Outputs (device, caller-owned; Wq and Wop may each be NULL but not both):
 *   Wq  uint8 [N][K/2] packed INT4;  Wop uint8 [N][K] GEMM operand (flags: RRS_OPERAND_I8 or not);
 *   w_scale f32 [N] = beta_n.
 * flags & RRS_W_PACKED4: Wop is instead the "decode4" packed W read by the decode GEMM, ceil(N/256)*256*K/2 bytes
 *   (half the HBM bytes of the one-code-per-byte operand; "different batch sizes"): contiguous 16 KiB tiles,
 *   tile (rb, kb) = rows [256 rb, 256 rb + 256) x K-block [128 kb, 128 kb + 128) at byte (rb * K/128 + kb) * 16384;
 *   inside a tile row r occupies 64 bytes at r * 64, its 32-code chunk c (codes j0 = 128 kb + 32 c ..) sits at
 *   r * 64 + 16 * (c ^ ((r >> 1) & 3)), and chunk byte b (0..15) = (q[j0+b] & 0xF) << 4 | (q[j0+16+b] & 0xF)
 *   (two's-complement nibbles).  Rows >= N are zero codes.
 * Offline helper: it takes a stream-ordered temporary (cudaMallocAsync, <= 256 MiB) for the rotated rows. */
rrs_status rrs_prepare_weights(const void* W, int32_t w_dtype, int64_t N, int64_t K, int32_t group,
                               const int32_t* perm, uint8_t* Wq, uint8_t* Wop, float* w_scale,
                               uint32_t flags, void* stream);

/* Runtime prologue:
 *   a1 X~ = X . H_K per token, exact in f64, rounded once to f32 (Eq. 4, R1-R3)
 *   a2 c_j = max over ALL T tokens of |X~_tj| (Eq. 1, R6)         -> chan_max (optional out)
 *   a3/a4 s_g = max_{j' in group g} c[perm[j']], 0 -> 1 (P:103(2), R5, R8)  -> s_group
 *   a5 Z = X~[:, perm] * fl(1/s_g) (Eq. 2, R9)
 *   a6 alpha_t = fl(max|Z_t| / 7), codes rint_even(fl(Z * fl(7/max))) (R9-R11) -> x_scale, Xq/Xop
 * X: device bf16 bits [T][K]; perm: device int32 [K];
 * outputs: Xq uint8 [T][K/2] (nullable), Xop uint8 [T][K] GEMM operand (nullable; flags as for
 *          rrs_prepare_weights), x_scale f32 [T],
 *          s_group f32 [K/group], chan_max f32 [K] (nullable).  Without chan_max the prefill prologue for
 *          K = 2^m (T > 64) is one cooperative launch that reduces the group maxima s_g directly (the max over
 *          tokens and the group's channels jointly, identical by construction); with chan_max it runs the rotate
 *          and quantise passes as two kernels.  Both give identical s_group, x_scale and codes.
 * ws: device scratch, 16-byte aligned, >= rrs_workspace_bytes(T, 1, K, group, 1) bytes (holds X~). */
rrs_status rrs_rotate_smooth_quant(const void* X, int32_t x_dtype, int64_t T, int64_t K, int32_t group,
                                   const int32_t* perm, uint8_t* Xq, uint8_t* Xop, float* x_scale,
                                   float* s_group, float* chan_max, void* ws, size_t ws_bytes, uint32_t flags,
                                   void* stream);

/* Fused grouped GEMM (fig:framework (3) P:103, P:109 step 3):
 *   P_g[t][n] = sum_{j' in g} q[t][j'] * qw[n][j']          (exact, in TMEM: FP32 or int32 by carrier)
 *   Y[t][n]   = out_scale * alpha_t * beta_n * sum_g s_g * P_g[t][n]   (f32 scale-accumulate)
 * out_scale = 1/K after rotation (R1).  flags & RRS_GEMM_PLAIN: per-channel A4W4 baseline
 * Y = out_scale * alpha_t * beta_n * sum_{all j'} q qw (s_group ignored, may be NULL).
 * flags & RRS_OPERAND_I8: operands are int8 codes, else E4M3 bytes (see the conventions above).
 * flags & RRS_GEMM_SUBCHANNEL (the second efficiency baseline of P:322): x_scale is
 *   alpha f32 [G][T] and w_scale beta f32 [G][N] (per token / per output row AND per group of `group` codes,
 *   sub-channel RTN), s_group is ignored: Y = out_scale * sum_g alpha_gt * beta_gn * P_g.  E4M3 operands only,
 *   N % 8 == 0, scales 16-byte aligned.
 * flags & RRS_GEMM_SWIGLU (LLaMA MLP; P:138 places RRS on the up/gate and down inputs): the N
 *   weight rows are interleaved gate/up pairs (row 2i = gate_i, row 2i+1 = up_i, N even) and Y receives
 *   bf16 [T][N/2] with Y[t][i] = bf16_rne(silu(y_2i) * y_2i+1), y = the f32 layer output above and
 *   silu(g) = g / (1 + e^-g) in f32 -- the input of the down_proj RRS layer, written once.  bf16 only.
 * flags & RRS_W_PACKED4 (decode regime, 1 <= T <= 64, group % 128 == 0): Xop is int8 codes [T][K] (the
 *   RRS_OPERAND_I8 activation carrier) and Wop the decode4-packed W of rrs_prepare_weights(RRS_W_PACKED4);
 *   same Y (any fixed FP32 order, R15), no PLAIN / SWIGLU / SUBCHANNEL.
 * Xop uint8 [T][K], x_scale f32 [T], s_group f32 [K/group], Wop uint8 [N][K], w_scale f32 [N];
 * Y [T][ldy] in y_dtype (bf16: round-to-nearest-even of the f32 result), ldy >= N, ldy % 8 == 0. */
rrs_status rrs_gemm(const uint8_t* Xop, const float* x_scale, const float* s_group, const uint8_t* Wop,
                    const float* w_scale, int64_t T, int64_t N, int64_t K, int32_t group, float out_scale,
                    uint32_t flags, void* Y, int32_t y_dtype, int64_t ldy, void* stream);

/* Whole layer = rrs_rotate_smooth_quant (into ws) + rrs_gemm with out_scale = 1/K.
 * comm == NULL: single GPU, Wop/w_scale hold all N rows.
 * flags & RRS_W_PACKED4 (comm == NULL, 1 <= T <= 64): Wop is the decode4-packed W; the prologue writes int8
 *   activation codes to ws and the decode GEMM streams the packed W (see rrs_gemm).
 * comm != NULL (column-parallel): Wop/w_scale hold THIS rank's N/world output rows
 *   [rank*N/world, (rank+1)*N/world); X is replicated; every rank runs the identical prologue; Y
 *   receives all N columns through an NCCL all-gather (any world >= 1; ws sized by rrs_workspace_bytes_comm).
 *   For T >= 1024 the GEMM runs in 256-row-aligned token slabs whose all-gathers run on an internal stream
 *   of the communicator, overlapping the next slab's GEMM; Y is complete in `stream` order on return.
 *   N_total % world == 0 required.
 * comm != NULL and flags & RRS_TOKEN_SHARDED (data parallel over tokens): X holds THIS
 *   rank's T tokens (T may differ between ranks, 0 included), Wop/w_scale hold all N_total rows, Y
 *   receives this rank's [T][N_total].  The runtime channel max is over ALL tokens of the call (Eq. 1
 *   P:90, R6): the rotate pass writes chan_max of the local tokens, one ncclAllReduce(MAX) of chan_max[K]
 *   f32 combines them, then every rank smooths and quantises with the same s_g -- codes, alpha_t and Y rows
 *   are bit-identical to one call on the concatenated tokens.  No output collective.  Every rank of comm
 *   must call it (collective). */
rrs_status rrs_linear(const void* X, int32_t x_dtype, int64_t T, int64_t K, int32_t group,
                      const int32_t* perm, const uint8_t* Wop, const float* w_scale, int64_t N_total,
                      void* Y, int32_t y_dtype, int64_t ldy, rrs_comm_t comm, void* ws, size_t ws_bytes,
                      uint32_t flags, void* stream);

/* The collective step of the column-parallel layer on its own: all-gather every rank's
 * Y shard [T][N_total/world] (contiguous, y_dtype) over NCCL and re-lay it out into Y[T][ldy]
 * (rank r's shard -> columns [r*N_total/world, (r+1)*N_total/world)).  ws as for rrs_linear. */
rrs_status rrs_allgather_columns(const void* Y_shard, int64_t T, int64_t N_total, int32_t y_dtype, void* Y,
                                 int64_t ldy, rrs_comm_t comm, void* ws, size_t ws_bytes, void* stream);

/* Communicator (NCCL over NVLink/NVSwitch).  torch.distributed only ferries the 128-byte id.  Collective calls
 * (rrs_linear / rrs_allgather_columns with a communicator) validate every argument before joining a collective, so
 * an argument error returns on the rank that made it; as with NCCL itself, arguments must agree across ranks or the
 * other ranks block in the collective. */
rrs_status rrs_comm_unique_id(uint8_t id[128]);
rrs_status rrs_comm_init(rrs_comm_t* comm, int32_t rank, int32_t world, const uint8_t id[128]);
rrs_status rrs_comm_destroy(rrs_comm_t comm);
int32_t rrs_comm_world(rrs_comm_t comm);
int32_t rrs_comm_rank(rrs_comm_t comm);

/* Test-only exports (same kernels, extra stores). */
/* X~ as f32 [T][K] (natural column order) and chan_max f32 [K] from the a1/a2 kernel. */
rrs_status rrs_debug_rotate(const void* X, int64_t T, int64_t K, float* Xr, float* chan_max, void* stream);
/* The column-parallel layer's re-layout step on its own (the step after ncclAllGather): gathered =
 * [world][T][n_shard] (rank-major, as ncclAllGather leaves it) -> Y[T][ldy] with rank r's shard in columns
 * [r n_shard, (r+1) n_shard).  Lets a single GPU emulate P ranks bit for bit (tests T3a). */
rrs_status rrs_debug_relayout(const void* gathered, int64_t T, int64_t n_shard, int32_t world, int32_t y_dtype,
                              void* Y, int64_t ldy, void* stream);
/* The tcgen05 GEMM's own group partials P[G][T][N] as int32 (read back from TMEM, same kernel). */
rrs_status rrs_debug_group_partials(const uint8_t* Xop, const uint8_t* Wop, int64_t T, int64_t N, int64_t K,
                                    int32_t group, int32_t* P, uint32_t flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* RRS_H_ */
