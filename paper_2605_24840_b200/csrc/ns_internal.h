// Internal declarations shared by the FP64 kernels (ns_fp64.cu) and the C-ABI host
// code (ns_api.cu).  Not part of the public ABI.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace nsr {

constexpr int kTile = 128;      // output tile edge (rows of P, rows of Q)
constexpr int kBK = 16;         // k-slab per pipeline stage: 16 doubles = one 128-B swizzle row
constexpr int kSPS = 2;         // 16-wide k-slabs per pipeline stage (one mbarrier wait per 2 slabs)
constexpr int kStages = 3;      // TMA ring depth (3 x 64 KB)
constexpr int kConsumerWarps = 8;
constexpr int kThreads = 32 * kConsumerWarps;         // 8 DMMA warps; warp 0 lane 0 also drives the TMA ring
constexpr int kStageBytes = kSPS * 2 * kTile * kBK * 8;   // A + B per stage = 64 KB
constexpr int kEpiPitch = kTile + 1;                  // staging row pitch (doubles), odd => conflict-free columns
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
// 64x64-tile variant (small / batched problems): 4 DMMA warps, 3 stages of 32 KB, 2 CTAs per SM
constexpr int kMaxFilterDeg = 4;   // general odd filters: degree <= 2*4+1 = 9 (ns_options_t.filter_c)
constexpr int k64Tile = 64;
#ifndef NS_K64_WARPS
#define NS_K64_WARPS 4
#endif
constexpr int k64Threads = 32 * NS_K64_WARPS;   // 4 DMMA warps (32x32 warp tiles) or 8 (32x16)
#ifndef NS_K64_STAGES
#define NS_K64_STAGES 2
#endif
constexpr int k64Stages = NS_K64_STAGES;
#ifndef NS_K64_SPS
#define NS_K64_SPS 2
#endif
constexpr int k64SPS = NS_K64_SPS;   // 16-wide k-slabs per stage of the 64-tile ring (k64Stages * k64SPS >= 4)
constexpr int k64StageBytes = k64SPS * 2 * k64Tile * kBK * 8;   // 32 KB at 2 slabs
#ifndef NS_K64_PAD
#define NS_K64_PAD 0
#endif
#ifndef NS_K64_MINB
#define NS_K64_MINB (k64Stages * k64SPS <= 4 ? 3 : 2)
#endif
constexpr int k64MinBlocks = NS_K64_MINB;   // CTAs per SM the register budget is sized for
constexpr int k64SmemBytes = k64Stages * k64StageBytes + 1024 + 256 + NS_K64_PAD;

// Per-problem device state (one per job).  Written only by ns_decide_kernel.
struct DevState {
  int32_t j;          // index of the current iterate X_j
  int32_t flags;      // NS_F_* bits
  int32_t done;       // 1 once a stop condition fired
  int32_t sw;         // mixed path: 1 once the low-precision phase hit the switch threshold
  double residual;    // r_j = ||X_j^2 - I||_F of the returned X
  double r_prev;      // r_{j-1}
  double trace;       // tr X_j
  int64_t cert;       // round((d - tr)/2)
  double sw_residual; // mixed path: low-precision residual at the switch
  int32_t sw_step;    // mixed path: j at the switch (-1 = none)
  int32_t spec;       // index j+1 of the iterate the decide at step j predicts to be final (0 = none)
  int32_t j_small;    // mixed path: first j with r_j/sqrt(d) < switch_tol in the low-precision phase (-1 = none);
                      // a conditioning proxy, min|x| of X_0 ~ 1.5^-(j_small - 3) (each NS step grows small |x| by 1.5)
  int32_t pad2;
};

// Per-problem scalar inputs (device copy).
struct JobParams {
  double s;
  double alpha;
  int32_t k;
  int32_t pad;
};

struct LoopParams {
  int d;               // true dimension
  int d_pad;           // padded dimension (multiple of kTile); workspace leading dim
  int max_steps;
  int tol_mode;        // 0 abs, 1 per sqrt(d)
  double tol;
  double switch_tol;   // mixed path: leave the low-precision phase when r/sqrt(d) < switch_tol
  int switch_at;       // mixed path, fixed-step mode: leave the low-precision phase at j == switch_at (-1: use switch_tol)
  int lowprec;         // 1 while running the low-precision phase of the mixed path
  double ca = 1.5;     // filter step coefficients (small fused kernel)
  double cb = -0.5;
};

// ---------------- re-anchor (ns_reanchor.cu) ----------------
// Device scalars of the conjugate-gradient solve |A|E + E|A| = F.
struct CgScalars {
  double rr;      // <R, R>
  double pw;      // <P, W>,  W = |A| P
  double alpha;
  double beta;
  double rr0;     // <R, R> of the initial residual
  double tol2;    // stop once rr <= tol2 * rr0 (relative residual tol, squared)
  int done;       // set by the scalar kernel; every later CG launch returns at once
  int iters;      // iterations performed
};
constexpr double kCgTol = 1e-6;      // re-anchor CG: stop at |R| <= kCgTol |R_0| (within the iteration cap)
constexpr int kCgRefineIters = 40;   // a solve that needed more iterations is followed by a second re-anchor pass
constexpr int kCgRefineJSmall = 12;
constexpr int kCgRefineMaxD = 2048;  // ... and every run with d <= this (the second pass is cheap there)  // ... and so is one whose |A| has condition ~ 1.5^(j_small - 3) > 30
constexpr int kEwBlocks = 148 * 8;   // fixed grid of the elementwise CG kernels (fixed-order partial sums)

// C = M - M^T, |A| = sym(M) planes; with partial: per-block ||C||_F^2 partials (n_partial of them)
cudaError_t launch_commutator(const double* M, double* C, void* abs_planes, int d_pad, cudaStream_t st,
                              bool tf32 = false, double* partial = nullptr, int* n_partial = nullptr);
cudaError_t launch_cg_init(const double* Fp, double* R, double* P, double* E, double* partial, int d_pad,
                           cudaStream_t st, int* n_partial);
cudaError_t launch_cg_pw(const double* P, const double* W, double* partial, int d_pad, cudaStream_t st,
                         const CgScalars* sc);
cudaError_t launch_cg_scalar(CgScalars* sc, const double* partial, int n_partial, int which, cudaStream_t st,
                             double tol2 = 0.0);
cudaError_t launch_cg_update(double* E, double* R, const double* P, const double* W, const CgScalars* sc,
                             double* partial, int d_pad, cudaStream_t st, int* n_partial);
cudaError_t launch_cg_direction(double* P, const double* R, const CgScalars* sc, void* p_planes, int d_pad,
                                cudaStream_t st, bool tf32 = false);
cudaError_t launch_apply_correction(double* X, const double* E, int d_pad, cudaStream_t st);

// Product kernel parameters: C_IJ = sum_k P[I,k] Q[J,k] on upper tiles (I <= J).
struct ProdParams {
  const int2* tiles;       // (I, J) tile list, n_tiles entries
  int n_tiles;
  int nk;                  // d_pad / kBK
  int d;                   // true dimension (identity mask in the residual)
  int ld;                  // d_pad
  long long job_stride;    // elements between consecutive jobs' matrices
  double* C;               // mode 0: Y ; mode 1: X_{j+1}
  const double* Xold;      // mode 1: X_j (read in the epilogue)
  double* partial;         // mode 0: residual partial per (job, tile); mode 1: trace partial per (job, I) on diag tiles
  const DevState* state;   // per-job state; CTA exits if state[job].done (nullptr = never)
  int mode;                // 0 = square/plain product + residual, 1 = NS update + trace
  double ca = 1.5;         // mode 1: X_{j+1} = ca X_j + cb X_j Y_j  (odd cubic filter step; NS: 1.5, -0.5)
  double cb = -0.5;
  double cc = 0.0;         // mode 1: + cc I (Horner steps of a general odd polynomial filter, ns_api.cu run_filter)
  // Peer-memory exchange (sharded path, modes 0/1): the epilogue also stores its tile, mirror and partial
  // into n_dst destination buffers (device arrays of base pointers, e.g. every rank's Y through CUDA IPC
  // peer mappings over NVLink); partial slots use the global tile index gt_off + blockIdx.x * gt_stride
  // in arrays of n_tiles_total per job.  n_dst = 0: local stores only.
  double* const* dst = nullptr;
  double* const* dst_part = nullptr;
  int n_dst = 0;
  int gt_off = 0, gt_stride = 1, n_tiles_total = 0;
  // batched: CTA row blockIdx.y runs job job_list[blockIdx.y] (rows >= *n_job_list exit); nullptr = job blockIdx.y
  const int* job_list = nullptr;
  const int* n_job_list = nullptr;
  // mode 0, batch 1: partial slot of CTA x is part_slot[x] (a sub-list of the tile list launched on its
  // own keeps the slots of the full list, so the decide's fixed-order sum is unchanged); nullptr = x
  const int* part_slot = nullptr;
  int diag_tri = 1;        // 64x64-tile kernel: diagonal tiles compute only their upper 8x8 blocks (NS_DIAG_TRI=0: full)
  int same_pq = 0;         // mode 0: P and Q are the same matrix (diagonal tiles then load one panel, not two)
  int dbg_sleep = 0;       // experiments (NS_P64_DBG_SLEEP, ns): every DMMA warp idles this long before its epilogue
  int dbg_int = 0;         // experiments (NS_P64_DBG_INT): ... and issues this many x4 extra integer instructions
  int remote_mirror = 1;   // peer-store epilogue: also store the mirrored tile into the other destinations (0: the
                           // receivers mirror remote tiles themselves, launch_mirror_remote; half the NVLink bytes)
};

// ---------------- mixed path (tcgen05 BF16x3, ns_mixed.cu) ----------------
constexpr int kMxBK = 64;                       // bf16 per k-block: 128 B = one swizzle row
constexpr int kMxStages = 3;
constexpr int kMxEpiWarps = 8;
constexpr int kMxEpiThreads = 32 * kMxEpiWarps;
constexpr int kMxThreads = 64 + kMxEpiThreads;  // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
#ifndef NS_MX_CHUNK_KB
#define NS_MX_CHUNK_KB 16
#endif
constexpr int kMxChunkKb = NS_MX_CHUNK_KB;      // k-blocks (x64) per FP32 accumulation chunk (x3 split terms)
constexpr int kMxSlab = kTile * kMxBK * 2;      // one 128 x 64 bf16 operand slab = 16 KB
constexpr int kMxStageBytes = 4 * kMxSlab;      // A_hi, A_lo, B_hi, B_lo = 64 KB
constexpr int kMxSmemBytes = kMxStages * kMxStageBytes + 1024 + 256;
// 2-SM variant (cta_group::2): a CTA pair computes a 256 x 128 tile with M=256 UMMAs; each CTA stages
// its own 128 rows of P and 64 of the 128 rows of Q (the two Q halves form one N=128 operand)
constexpr int kMx2Stages = 4;
constexpr int kMx2SlabA = kTile * kMxBK * 2;     // 128 x 64 bf16 = 16 KB
constexpr int kMx2SlabB = 64 * kMxBK * 2;        // 64 x 64 bf16 = 8 KB
constexpr int kMx2StageBytes = 2 * kMx2SlabA + 2 * kMx2SlabB;   // 48 KB per CTA
constexpr int kMx2SmemBytes = kMx2Stages * kMx2StageBytes + 1024 + 256;

// C_IJ = sum over the 3 split terms of P'_I Q'_J^T with P' = [P_hi P_lo P_hi], Q' = [Q_lo Q_hi Q_hi]
// (small terms first), FP32 accumulation in TMEM.  Planes: [job][hi|lo][d_pad][d_pad] bf16.
struct MxParams {
  const int2* tiles;
  int n_tiles;
  int nkb;                 // d_pad / kMxBK
  int d;
  int ld;                  // d_pad
  long long job_stride;    // FP64 elements between jobs' matrices
  double* C;               // FP64 output (mode 0: Y, 1: X_{j+1}, 2: W dense)
  const double* Xold;      // mode 1
  void* Cplanes;           // hi/lo planes of C (bf16 or tf32-as-fp32; modes 0, 1), nullptr = skip
  double* partial;         // mode 0 residual partial per tile; mode 1 trace partial per diag block
  const DevState* state;
  int mode;                // 0 square (+res, mirror), 1 update (+trace, mirror), 2 dense tile (no mirror)
  int tf32 = 0;            // 0: BF16x3 (kind::f16), 1: TF32x3 (kind::tf32); nkb = d_pad / (tf32 ? 32 : 64)
  unsigned long long* trace = nullptr;   // diagnostics: per-CTA %globaltimer stamps (start, mainloop done, end)
  const int* skip = nullptr;             // CG operator products: return at once if *skip (solve converged)
};

cudaError_t launch_split_planes(const double* X, void* planes, int d_pad, int batch, cudaStream_t st,
                                bool tf32 = false);
cudaError_t launch_mx_product(const CUtensorMap& tmP, const CUtensorMap& tmQ, const MxParams& p, int batch,
                              cudaStream_t st);
// 2-SM launch: p.tiles holds (I2, J) pairs (256-row block, 128-column block), p.n_tiles = 2 x pairs;
// tmQ must be a 64-row-box map of the Q planes
cudaError_t launch_mx2_product(const CUtensorMap& tmP, const CUtensorMap& tmQ64, const MxParams& p, int batch,
                               cudaStream_t st);

// Host-side launchers (ns_fp64.cu).
cudaError_t launch_init(const double* H, long long ldh, long long h_stride, double* X, const JobParams* jobs,
                        int d, int d_pad, int batch, cudaStream_t st, int rb0 = 0, int rb1 = -1);   // 64-row blocks [rb0, rb1)
cudaError_t launch_trace_partials(const double* X, int d, int d_pad, int batch, double* tr_partial,
                                  cudaStream_t st, int job_stride = 0);
// Raise a kernel's dynamic shared-memory limit once per device: `mask` is that kernel's static set of
// devices already configured (one process may drive several GPUs; the setting is per device).
template <typename F>
inline void smem_attr(F* fn, int bytes, unsigned long long& mask) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (mask & bit) return;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) == cudaSuccess) mask |= bit;
}

cudaError_t launch_product64(const CUtensorMap& tmP, const CUtensorMap& tmQ, const ProdParams& p, int batch,
                             cudaStream_t st);
cudaError_t launch_product(const CUtensorMap& tmP, const CUtensorMap& tmQ, const ProdParams& p, int batch,
                           cudaStream_t st);
cudaError_t launch_decide(DevState* state, const JobParams* jobs, const double* res_partial, int n_tiles,
                          const double* tr_partial, int n_diag, LoopParams lp, int batch, int* n_active,
                          cudaStream_t st, const double* res_ranks = nullptr, int nranks = 0);

// ---------------- small-d fused path (ns_small.cu): d <= 96, whole loop in one CTA per problem ----------------
int small_dpad(int d);
int small_trace_read(unsigned long long* out, int n);                    // NS_SMALL_TRACE diagnostics
int p64_trace_set(unsigned long long* buf, unsigned long long cap);      // NS_P64_TRACE diagnostics
cudaError_t launch_small(const double* H, long long ldh, long long h_stride, const JobParams* jobs, JobParams job0,
                         LoopParams lp, double* R, long long ldr, long long r_stride, DevState* state, int batch,
                         cudaStream_t st);

// ---------------- Algorithm 1 outer loop on the rotated quartic (ns_outer.cu), d <= 64 ----------------
struct OuterParams {
  int m;              // Newton–Schulz depth of the filter (0 = exact reflector)
  int max_iters;
  double eta;         // fixed outer step size
  double grad_tol;
  int policy;         // shift policy (alg:ssr step 4): 0 midpoint, 1 damped midpoint, 2 reuse/refresh
  int pad;
  double damp;        // damped: weight of the previous shift
  double clip;        // damped: clip into [lk + clip gap, lk1 - clip gap]
  double reuse_margin;  // reuse/refresh: keep the previous shift while its margin exceeds this
  double eps;         // admissibility: stop unless the chosen shift's estimated margin exceeds eps
};
struct OuterResult {
  int iters;
  int morse_index;
  int success;
  int stop_reason;    // 0 ||g|| <= grad_tol, 1 budget, 2 inadmissible shift
  double grad_norm;
  int refreshes;      // iterations that took the fresh midpoint
  int pad;
  double s_last;      // last shift used in an update (NaN when none)
};
cudaError_t launch_outer(const double* Q, int d, const int* k, const double* x0, OuterParams p, double* xout,
                         OuterResult* res, int nruns, cudaStream_t st);

// ---------------- Ozaki-split FP64 products on INT8 tensor cores (ns_ozaki.cu) ----------------
constexpr int kOzSlices = 7;                           // balanced base-256 int8 digits per entry (54 bits)
// digit-pair groups kept per launch (OzParams.groups, pairs s + t < groups): 7 keeps the 28 pairs of weight
// >= 2^-48; 8 adds the six pairs of weight 2^-56 (+21% MACs; the eighth INT32 group fills TMEM columns
// 448..511), which lowers the dropped-pair residual floor from ~1.5e-15 d to ~4e-17 d (FP64 DMMA: 3e-17 d)
constexpr int kOzChunkKb = 256;                        // k-blocks (x64) per INT32 chunk: exact for any d
constexpr int kOzMaxD = 65536;
#ifndef NS_OZ_KH
#define NS_OZ_KH 64
#endif
// K bytes per ring stage: 64 (64-byte swizzle, 2 stages of 84 KB; default) or 32 (one UMMA K step,
// 32-byte swizzle, 4 stages of 42 KB, -DNS_OZ_KH=32).  The operand feed (L2 -> SMEM over TMA) and the
// tensor pipe take about equally long per k-block here (32 ms each for a d = 16384 product when
// measured alone, 39 ms together), so finer stages were tried for a better overlap: measured A/B they
// are 12% slower (twice the TMA requests of half the width).
constexpr int kOzKH = NS_OZ_KH;
constexpr int kOzStages = kOzKH == 32 ? 4 : 2;
constexpr int kOzThreads = 320;                        // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue
constexpr int kOzSlabA = kTile * kOzKH;                // 128 rows x kOzKH int8
constexpr int kOzSlabB = 64 * kOzKH;                   // 64 rows x kOzKH int8
constexpr int kOzStageBytes = kOzSlices * (kOzSlabA + kOzSlabB);
constexpr int kOzSmemBytes = kOzStages * kOzStageBytes + 1024 + 256 + 8 * 32 * 17 * 8;   // + epilogue staging

struct OzParams {
  const int2* tiles;       // (I: 128-row block, J2: 64-column block)
  int n_tiles;
  int nkb;                 // d_pad / 64
  int d;
  int ld;                  // d_pad
  long long job_stride;
  double* C;
  const double* Xold;      // mode 1
  const int* expP;         // row exponents of P (per job, d_pad)
  const int* expQ;         // row exponents of Q
  double* partial;         // mode 0: per tile; mode 1: per 64-column block J2 (2n entries per job)
  const DevState* state;
  int mode;                // 0 square (+res, mirror), 1 update (+trace, mirror), 2 dense
  double ca = 1.5;
  double cb = -0.5;
  double cc = 0.0;         // mode 1: + cc I on the diagonal (general odd polynomial filters)
  int kb0 = 0;             // first k-block of this launch (K segments, see launch_ozaki_product)
  int pm = 0;              // 0 whole K; K segments: 1 first (C = raw sums), 2 middle (C += raw), 3 last (C + raw -> epilogue)
  int dbg = 0;             // experiments only (NS_OZ_DBG): 1 = stream operands without issuing the UMMAs
  int groups = 7;          // digit-pair groups kept (7 or 8, see kOzSlices)
};
constexpr int kOzBadRow = 1 << 20;   // row exponent marking a non-finite row (its products become NaN)
constexpr int kOzSegKb = 256;   // k-blocks per K segment (K = 16384): one launch per segment for larger d
bool use_oz_mc();   // Ozaki products on CTA clusters of 2 (A digits multicast); NS_OZ_MC=0 disables
cudaError_t launch_ozaki_slice(const double* X, int8_t* slices, int* expo, int d_pad, int batch, cudaStream_t st);
cudaError_t launch_ozaki_product(const CUtensorMap& tmA, const CUtensorMap& tmB, const OzParams& p, int batch,
                                 cudaStream_t st);

// ---------------- shift/scale setup (ns_setup.cu) ----------------
cudaError_t launch_scale_bound(const double* H, long long ldh, int d, double s, double* part, double* out,
                               cudaStream_t st);

// ---------------- sharded path (ns_shard.cu) ----------------
cudaError_t launch_pack_tiles(const double* M, const int2* my_tiles, int n_my, double* send, int d_pad,
                              cudaStream_t st);
cudaError_t launch_unpack_tiles(double* M, const int2* all_tiles, int n_tiles, const double* recv_chunk, int cs,
                                int slot0, int nranks, int my_rank, int d_pad, cudaStream_t st);
cudaError_t launch_shard_sum(const double* v, int n, double* out, cudaStream_t st);
// R (rows row0 .. row0 + rows - 1 of the returned iterate; rows < 0: to d) <- X_steps
cudaError_t launch_copy_out(const double* Xa, const double* Xb, int d, int d_pad, const DevState* state,
                            double* R, long long ldr, long long r_stride, int batch, cudaStream_t st, int row0 = 0,
                            int rows = -1);
// Receiver-side mirror (sharded path, remote_mirror = 0): for every off-diagonal upper tile of the global
// list NOT computed by my_rank (t % nranks != my_rank), M[J-block][I-block] <- M[I-block][J-block]^T.
cudaError_t launch_mirror_remote(double* M, const int2* all_tiles, int n_tiles, int nranks, int my_rank, int d_pad,
                                 cudaStream_t st);
// Block-row input (sharded rows entry): rows [r0, r1) of H (local buffer H_rows, leading dimension ldh, only
// elements j >= i read) -> X_0 = (H - sI)/alpha elements (i, j) and (j, i) into every destination X in dst[0..n_dst)
// (device array of base pointers, d_pad x d_pad).  Elements of other ranks' rows and the padding are not written.
cudaError_t launch_init_rows(const double* H_rows, long long ldh, long long r0, long long r1, double* const* dst,
                             int n_dst, double s, double alpha, int d, int d_pad, cudaStream_t st);
cudaError_t launch_zero_state(DevState* state, int batch, int* n_active, cudaStream_t st);
// If state->spec == jn: copy X (d x d inside d_pad) to R (device-accessible pinned host memory, leading
// dimension ldr) -- the speculative result copy of the host entry (ns_api.cu run_loop)
cudaError_t launch_spec_copy(const DevState* state, int jn, const double* X, int d, int d_pad, double* R,
                             long long ldr, cudaStream_t st);
// list[0..*n_list) = the jobs with !state[job].done in ascending order (one CTA, stable)
cudaError_t launch_compact(const DevState* state, int batch, int* list, int* n_list, cudaStream_t st);

}  // namespace nsr
