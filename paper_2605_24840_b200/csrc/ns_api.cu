// C-ABI entry points of libnsreflector.so (declared in include/nsreflector.h).
//
// Host responsibilities only: argument validation, workspace carve-up, TMA tensor-map
// encoding, and the step loop that enqueues the device kernels (ns_fp64.cu).  The stop
// decision is taken on the device (ns_decide_kernel); the host enqueues a bounded number
// of steps ahead and only reads a 4-byte "problems still running" counter, so kernels
// enqueued after convergence exit immediately.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>
#include <algorithm>
#include <array>

#include "../../include/nsreflector.h"
#include "ns_internal.h"
#include <nccl.h>

using namespace nsr;

namespace {

thread_local std::string g_last_error;

ns_status_t fail(ns_status_t st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define NS_CUDA(x)                                                                          \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess)                                                                  \
      return fail(NS_ERR_CUDA, "%s failed: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                                \
  } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Layout {
  int d = 0, d_pad = 0, n = 0, n_tiles = 0;
  long long batch = 1;
  bool mixed = false;
  size_t off_xa = 0, off_xb = 0, off_y = 0, off_res = 0, off_tr = 0, off_tiles = 0, off_jobs = 0,
         off_state = 0, off_active = 0, off_px = 0, off_py = 0, off_full = 0, off_pxb = 0, off_ahat = 0,
         off_r = 0, off_p = 0, off_cgpart = 0, off_cgsc = 0, off_ozx = 0, off_ozy = 0, off_oex = 0, off_oey = 0,
         off_ores = 0, off_otr = 0, off_otiles = 0, off_ptiles = 0, off_pfull = 0, off_jlist = 0, off_tperm = 0,
         off_tslot = 0, total = 0;
};

Layout make_layout(int64_t d, int64_t batch, bool mixed = false, bool ozaki = false, bool tf32 = false) {
  Layout L;
  L.d = static_cast<int>(d);
  L.d_pad = static_cast<int>((d + kTile - 1) / kTile * kTile);
  L.n = L.d_pad / kTile;
  L.n_tiles = L.n * (L.n + 1) / 2;
  L.batch = batch;
  const size_t mat = (size_t)L.d_pad * (size_t)L.d_pad * sizeof(double) * (size_t)batch;
  size_t o = 0;
  L.off_xa = o; o = align256(o + mat);
  L.off_xb = o; o = align256(o + mat);
  L.off_y = o; o = align256(o + mat);
  // residual / trace partials and the tile list sized for 64-tiles too (use_tile64)
  const size_t n64 = 2 * (size_t)L.n, nt_max = std::max<size_t>(L.n_tiles, n64 * (n64 + 1) / 2);
  L.off_res = o; o = align256(o + sizeof(double) * nt_max * batch);
  L.off_tr = o; o = align256(o + sizeof(double) * n64 * batch);
  L.off_tiles = o; o = align256(o + sizeof(int2) * nt_max);
  L.off_tperm = o; o = align256(o + sizeof(int2) * nt_max);   // first square of the host entry: tiles by H chunk
  L.off_tslot = o; o = align256(o + sizeof(int) * nt_max);    // ... and their partial slots
  L.off_jobs = o; o = align256(o + sizeof(JobParams) * (size_t)batch);
  L.off_state = o; o = align256(o + sizeof(DevState) * (size_t)batch);
  L.off_active = o; o = align256(o + 256);
  L.off_jlist = o; o = align256(o + sizeof(int) * ((size_t)batch + 1));   // active-job list + its count
  L.off_full = o; o = align256(o + sizeof(int2) * (size_t)L.n * L.n);   // full tile list (dense products)
  L.mixed = mixed;
  if (ozaki) {
    const size_t nn = (size_t)L.d_pad * L.d_pad;
    L.off_ozx = o; o = align256(o + nn * kOzSlices * (size_t)batch);     // int8 slices of X_j
    L.off_ozy = o; o = align256(o + nn * kOzSlices * (size_t)batch);     // int8 slices of Y_j
    L.off_oex = o; o = align256(o + sizeof(int) * (size_t)L.d_pad * batch);
    L.off_oey = o; o = align256(o + sizeof(int) * (size_t)L.d_pad * batch);
    L.off_ores = o; o = align256(o + sizeof(double) * (size_t)L.n * (L.n + 1) * batch);   // 128x64 tiles
    L.off_otr = o; o = align256(o + sizeof(double) * (size_t)2 * L.n * batch);
    L.off_otiles = o; o = align256(o + sizeof(int2) * (size_t)2 * L.n * L.n);           // sym or full 128x64 list
  }
  if (mixed) {
    const size_t planes = (size_t)L.d_pad * L.d_pad * 2 * (tf32 ? 4 : 2) * (size_t)batch;   // hi + lo
    L.off_px = o; o = align256(o + planes);     // bf16 hi/lo planes of X_j (even j) / CG direction P
    L.off_pxb = o; o = align256(o + planes);    // bf16 hi/lo planes of X_j (odd j)
    L.off_py = o; o = align256(o + planes);     // bf16 hi/lo planes of Y / |A|
    L.off_ahat = o; o = align256(o + mat);      // A = X_0 kept in FP64 for the re-anchor; later E
    L.off_r = o; o = align256(o + mat);         // CG residual R
    L.off_p = o; o = align256(o + mat);         // CG direction P
    const int nb = L.d_pad / 32;
    const size_t npart = std::max<size_t>((size_t)nb * (nb + 1) / 2, (size_t)kEwBlocks);
    L.off_cgpart = o; o = align256(o + sizeof(double) * npart);
    L.off_cgsc = o; o = align256(o + sizeof(CgScalars));
    L.off_ptiles = o; o = align256(o + sizeof(int2) * (size_t)L.n * L.n);   // 2-SM pair list, upper
    L.off_pfull = o; o = align256(o + sizeof(int2) * (size_t)L.n * L.n);    // 2-SM pair list, dense
  }
  L.total = o;
  return L;
}

// 128 x 64 tiles (I: 128-row block, J2: 64-column block).  Symmetric: every tile touching the upper
// triangle (J2*64 + 63 >= I*128), L2-grouped like make_tiles; dense: all.
std::vector<int2> make_tiles_oz(int n, bool sym) {
  std::vector<int2> v;
  static const int G = [] {
    const char* e = getenv("NS_TILE_GROUP_OZ");   // experiment knob (super-block edge in 128-row blocks)
    const int g = e ? atoi(e) : 0;
    return g > 0 ? g : 12;
  }();
  for (int SI = 0; SI < n; SI += G)
    for (int SJ = sym ? 2 * SI : 0; SJ < 2 * n; SJ += 2 * G)
      for (int I = SI; I < std::min(SI + G, n); ++I)
        for (int J2 = std::max(SJ, sym ? 2 * I : 0); J2 < std::min(SJ + 2 * G, 2 * n); ++J2) v.push_back(make_int2(I, J2));
  return v;
}

// Tile pairs for the 2-SM split-precision kernel: (I2, J) = rows [256 I2, +256) x cols [128 J, +128);
// sym: only pairs touching the upper triangle (J >= 2 I2).  Super-blocks as in make_tiles.
std::vector<int2> make_tiles_pairs(int n, bool sym) {
  const int n2 = (n + 1) / 2, G = 8;
  std::vector<int2> v;
  for (int SI = 0; SI < n2; SI += G / 2)
    for (int SJ = sym ? 2 * SI : 0; SJ < n; SJ += G)
      for (int I2 = SI; I2 < std::min(SI + G / 2, n2); ++I2)
        for (int J = std::max(SJ, sym ? 2 * I2 : 0); J < std::min(SJ + G, n); ++J) v.push_back(make_int2(I2, J));
  return v;
}

// Diagnostics: when set, the 2-SM split-precision kernel launched by ns_symm_product records per-CTA
// %globaltimer stamps (start, accumulators done, end, SM id) -- tools/mx_timeline.py.
unsigned long long* g_mx_trace = nullptr;

// 2-SM (cta_group::2) split-precision products on by default; NS_MX2=0 selects the one-SM kernel.
bool use_mx2() {
  static const bool on = [] {
    const char* e = getenv("NS_MX2");
    return !(e && e[0] == '0');
  }();
  return on;
}

std::vector<int2> make_tiles_full(int n) {
  std::vector<int2> v;
  v.reserve((size_t)n * n);
  static const int G = [] {
    const char* e = getenv("NS_TILE_GROUP_FULL");   // experiment knob, like NS_TILE_GROUP
    const int g = e ? atoi(e) : 0;
    return g > 0 ? g : 6;
  }();
  for (int SI = 0; SI < n; SI += G)
    for (int SJ = 0; SJ < n; SJ += G)
      for (int I = SI; I < std::min(SI + G, n); ++I)
        for (int J = SJ; J < std::min(SJ + G, n); ++J) v.push_back(make_int2(I, J));
  return v;
}

// Upper-triangle tile order: super-blocks of G x G tiles (row-major over the upper
// triangle of super-blocks), row-major inside each.  Co-resident CTAs then share a
// few dozen row panels, so each k-slab of a panel is fetched from HBM about once per
// wave and re-read from L2 by the other CTAs.
int tile_group() {
  static int g = [] {
    const char* e = getenv("NS_TILE_GROUP");   // experiment knob: super-block edge of the tile order
    int v = e ? atoi(e) : 0;
    return v > 0 ? v : 8;
  }();
  return g;
}

std::vector<int2> make_tiles(int n) {
  const int G = tile_group();
  std::vector<int2> v;
  v.reserve((size_t)n * (n + 1) / 2);
  for (int SI = 0; SI < n; SI += G)
    for (int SJ = SI; SJ < n; SJ += G)
      for (int I = SI; I < std::min(SI + G, n); ++I)
        for (int J = std::max(SJ, I); J < std::min(SJ + G, n); ++J) v.push_back(make_int2(I, J));
  return v;
}

// Ozaki tile list and the number of per-tile residual partials it yields: 128x128 tiles walked by CTA
// clusters of 2 (each CTA one 64-column half, A digits multicast; default) or 128x64 single-CTA tiles.
std::vector<int2> oz_tile_list(int n, bool sym) {
  return use_oz_mc() ? (sym ? make_tiles(n) : make_tiles_full(n)) : make_tiles_oz(n, sym);
}
int oz_partials(const std::vector<int2>& ot) { return (use_oz_mc() ? 2 : 1) * (int)ot.size(); }

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 3-D map over `batch` row-major d_pad x d_pad FP64 matrices; box = 16 (k) x 128 (rows) x 1,
// 128-byte swizzle (the consumer's fragment addressing assumes exactly this pattern).
ns_status_t encode_map(CUtensorMap* m, const double* base, int d_pad, long long batch, int box_rows = kTile) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d_pad, (cuuint64_t)d_pad, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)d_pad * 8, (cuuint64_t)d_pad * (cuuint64_t)d_pad * 8};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return NS_OK;
}

// 3-D map over `nplanes` row-major d_pad x d_pad int8 slices; box = 64 (k) x rows x 1, 64-byte swizzle.
ns_status_t encode_map_i8(CUtensorMap* m, const int8_t* base, int d_pad, long long nplanes, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)d_pad, (cuuint64_t)d_pad, (cuuint64_t)nplanes};
  cuuint64_t strides[2] = {(cuuint64_t)d_pad, (cuuint64_t)d_pad * (cuuint64_t)d_pad};
  cuuint32_t box[3] = {(cuuint32_t)kOzKH, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, kOzKH == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled (int8) failed (%d)", (int)r);
  return NS_OK;
}

// 3-D map over `nplanes` row-major d_pad x d_pad BF16 planes; box = 64 (k) x 128 (rows) x 1, 128-B swizzle
// (the layout the UMMA shared-memory descriptors in ns_mixed.cu describe).
ns_status_t encode_map_bf16(CUtensorMap* m, const void* base, int d_pad, long long nplanes, bool tf32 = false,
                            int box_rows = kTile) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  const cuuint64_t esz = tf32 ? 4 : 2;
  cuuint64_t dims[3] = {(cuuint64_t)d_pad, (cuuint64_t)d_pad, (cuuint64_t)nplanes};
  cuuint64_t strides[2] = {(cuuint64_t)d_pad * esz, (cuuint64_t)d_pad * (cuuint64_t)d_pad * esz};
  cuuint32_t box[3] = {(cuuint32_t)(128 / esz), (cuuint32_t)box_rows, 1};   // 128-byte rows: 64 bf16 or 32 tf32
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, tf32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                   const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NS_ERR_CUDA, "cuTensorMapEncodeTiled (bf16) failed (%d)", (int)r);
  return NS_OK;
}

struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  ns_profile_t acc{};
  cudaEvent_t get(size_t i) {
    while (pool.size() <= i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[i];
  }
};

Profiler& prof() {
  static thread_local Profiler p;
  return p;
}

// Split-precision / Ozaki product launches, timed when profiling is on (bench.py's executed-arithmetic
// rooflines).  kind: 0/1 = BF16x3 symmetric / dense tile lists, 2/3 = Ozaki symmetric / dense.
struct XProf {
  struct Rec {
    cudaEvent_t a, b;
    int kind;
    double work;
  };
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<Rec> recs;
  cudaEvent_t ev() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};
XProf& xprof() {
  static thread_local XProf x;
  return x;
}
template <class F>
cudaError_t xtimed(cudaStream_t st, int kind, double work, F&& launch) {
  if (!prof().on) return launch();
  XProf& x = xprof();
  cudaEvent_t a = x.ev(), b = x.ev();
  cudaEventRecord(a, st);
  const cudaError_t e = launch();
  cudaEventRecord(b, st);
  x.recs.push_back({a, b, kind, work});
  return e;
}
// After the call's final stream synchronisation: add the launches that did work to the accumulators.
void xprof_flush() {
  XProf& x = xprof();
  if (x.recs.empty()) return;
  std::vector<float> ms(x.recs.size(), 0.f);
  float mx[4] = {0.f, 0.f, 0.f, 0.f};
  for (size_t i = 0; i < x.recs.size(); ++i) {
    cudaEventElapsedTime(&ms[i], x.recs[i].a, x.recs[i].b);
    mx[x.recs[i].kind] = std::max(mx[x.recs[i].kind], ms[i]);
  }
  ns_profile_t& acc = prof().acc;
  for (size_t i = 0; i < x.recs.size(); ++i) {
    const XProf::Rec& r = x.recs[i];
    if (ms[i] < 0.25f * mx[r.kind]) continue;        // exited at once (past a stop / converged CG)
    if (r.kind < 2) {
      acc.n_lowp += 1;
      acc.ms_lowp += ms[i];
      acc.lowp_flops += r.work;
    } else {
      acc.n_oz += 1;
      acc.ms_oz += ms[i];
      acc.oz_ops += r.work;
    }
  }
  x.recs.clear();
  x.used = 0;
}

struct HostRing {
  int* slots = nullptr;
  DevState* pstate = nullptr;   // pinned, mapped landing slot for single-problem results
  DevState* dstate = nullptr;   // its device alias: the fused small-d kernel writes the result there
  cudaEvent_t ev[16];
  bool ok = false;
};

HostRing& ring() {   // per host thread and device (events and mapped memory belong to one device)
  static thread_local HostRing rings[32];
  int dev = 0;
  cudaGetDevice(&dev);
  HostRing& r = rings[dev & 31];
  if (!r.ok) {
    if (cudaHostAlloc(&r.slots, 16 * sizeof(int), cudaHostAllocDefault) != cudaSuccess) return r;
    if (cudaHostAlloc(&r.pstate, sizeof(DevState), cudaHostAllocMapped) != cudaSuccess) r.pstate = nullptr;
    if (r.pstate && cudaHostGetDevicePointer(reinterpret_cast<void**>(&r.dstate), r.pstate, 0) != cudaSuccess)
      r.dstate = nullptr;
    for (int i = 0; i < 16; ++i) cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming);
    r.ok = true;
  }
  return r;
}

// Relative residual at which the re-anchor's CG solve stops (remaining launches of the capped loop
// return at once); NS_CG_TOL overrides (experiments)
double cg_tol() {
  static const double v = [] {
    const char* e = getenv("NS_CG_TOL");
    return e ? atof(e) : kCgTol;
  }();
  return v;
}

// Side stream + events of the speculative result copy (host entry, one per thread)
struct SpecCtx {
  cudaStream_t side = nullptr;
  cudaEvent_t upd = nullptr, cp[2] = {nullptr, nullptr}, end = nullptr, chunk[8] = {};
  bool ok = false;
};

SpecCtx& spec_ctx() {   // per host thread and device
  static thread_local SpecCtx ctxs[32];
  int dev = 0;
  cudaGetDevice(&dev);
  SpecCtx& c = ctxs[dev & 31];
  if (!c.ok) {
    if (cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking) != cudaSuccess) return c;
    cudaEventCreateWithFlags(&c.upd, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c.cp[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c.cp[1], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c.end, cudaEventDisableTiming);
    for (cudaEvent_t& e : c.chunk) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    c.ok = true;
  }
  return c;
}

ns_status_t check_common(int64_t d, int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec) {
  if (d < 1 || d > 65536) return fail(NS_ERR_INVALID_ARG, "d must be in [1, 65536], got %lld", (long long)d);
  if (max_steps < 0) return fail(NS_ERR_INVALID_ARG, "max_steps must be >= 0");
  if (!(tol >= 0.0) || !std::isfinite(tol)) return fail(NS_ERR_INVALID_ARG, "tol must be finite and >= 0");
  if (tm != NS_TOL_ABS && tm != NS_TOL_PER_SQRT_D) return fail(NS_ERR_INVALID_ARG, "bad tolerance mode");
  if (prec != NS_PREC_FP64 && prec != NS_PREC_MIXED_BF16X3 && prec != NS_PREC_MIXED_TF32X3 &&
      prec != NS_PREC_FP64_OZAKI)
    return fail(NS_ERR_INVALID_ARG, "bad precision");
  return NS_OK;
}

struct Opts {
  double switch_tol = 1e-3;   // reading C16b: 10x above the split-precision residual's noise floor
  int cg_iters = 512;             // cap; the solve stops at the relative residual cg_tol()
  int stop_at_switch = 0;
  int lookahead = 0;
  int polish = 2;                 // mixed path: 0 = all FP64 DMMA, 1 = all Ozaki INT8, 2 = Ozaki re-anchor + DMMA polish
  double ca = 1.5, cb = -0.5;
  double cz[kMaxFilterDeg - 1] = {0.0, 0.0, 0.0};   // coefficients of X^5, X^7, X^9 (general filters, run_filter)
  bool general_filter() const {
    for (double v : cz)
      if (v != 0.0) return true;
    return false;
  }
  // host entry: the caller's pinned R (device-accessible address) for the speculative result copy;
  // run_loop sets *spec_hit when R already holds the returned iterate
  double* spec_R = nullptr;
  long long spec_ldr = 0;
  bool* spec_hit = nullptr;
  // host entry, one problem: H is still on the host (h_host, leading dimension h_ldh); run_loop stages
  // it in row chunks on the side stream and starts the first square's tiles as their rows arrive
  const double* h_host = nullptr;
  long long h_ldh = 0;
};

Opts to_opts(const ns_options_t* o) {
  Opts r;
  if (o) {
    r.switch_tol = o->switch_tol;
    r.cg_iters = o->cg_iters;
    r.stop_at_switch = o->stop_at_switch;
    r.lookahead = o->lookahead;
    r.polish = o->polish;
    r.ca = o->filter_a;
    r.cb = o->filter_b;
    for (int i = 0; i < kMaxFilterDeg - 1; ++i) r.cz[i] = o->filter_c[i];
  }
  return r;
}

// 64x64 or 128x128 product tiles for the FP64 step loop.  Wave model: a 128-tile costs T per SM
// (one CTA per SM); three 64-tile CTAs share an SM and finish a wave of 3 x n_SM tiles in ~0.75 T.
// 64-tiles are taken when they need >= 5% less time (small d, batches, and sizes where 128-tiles
// leave a mostly empty last wave -- d = 3000: 26.5 ms vs 18.1 ms, d = 8192: -6.7%), else 128-tiles
// (d = 16384: 56 waves either way; the 128 kernel is the profiled headline kernel).
// NS_TILE64=0/1 forces one kind (experiments).
bool use_tile64(int d_pad, long long batch) {
  static const int force = [] {
    const char* e = getenv("NS_TILE64");
    return e ? atoi(e) : -1;
  }();
  if (force == 0 || force == 1) return force == 1;
  static int n_sm = 0;
  if (n_sm == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n_sm <= 0) n_sm = 148;
  }
  const long long n = d_pad / kTile, m = d_pad / k64Tile;
  const long long t128 = n * (n + 1) / 2 * batch, t64 = m * (m + 1) / 2 * batch;
  const double w128 = (double)((t128 + n_sm - 1) / n_sm);
  const double w64 = 0.75 * (double)((t64 + 3 * n_sm - 1) / (3 * n_sm));
  return w64 <= 0.95 * w128;
}

// The step loop shared by the single, host and batched entry points.  H: batch matrices
// at H + b*h_stride (ld ldh).  R likewise.  Returns per-job states in `states`.
ns_status_t run_loop(const Layout& L, uint8_t* ws, const double* H, long long ldh, long long h_stride,
                     const std::vector<JobParams>& jobs, int32_t max_steps, double tol, ns_tolmode_t tm, double* R,
                     long long ldr, long long r_stride, cudaStream_t st, std::vector<DevState>& states,
                     int* launches, const Opts& opt = Opts{}) {
  const int batch = (int)L.batch;
  double* Xa = reinterpret_cast<double*>(ws + L.off_xa);
  double* Xb = reinterpret_cast<double*>(ws + L.off_xb);
  double* Y = reinterpret_cast<double*>(ws + L.off_y);
  double* res = reinterpret_cast<double*>(ws + L.off_res);
  double* trp = reinterpret_cast<double*>(ws + L.off_tr);
  int2* tiles = reinterpret_cast<int2*>(ws + L.off_tiles);
  JobParams* djobs = reinterpret_cast<JobParams*>(ws + L.off_jobs);
  DevState* state = reinterpret_cast<DevState*>(ws + L.off_state);
  int* n_active = reinterpret_cast<int*>(ws + L.off_active);

  HostRing& rg = ring();
  if (!rg.ok) return fail(NS_ERR_CUDA, "pinned status ring allocation failed");

  if (small_dpad(L.d) != 0) {
    // d <= 96: one fused kernel (one CTA per problem runs the whole loop in shared memory); a single
    // problem passes its scalars by value and returns its state through pinned memory (no staging).
    LoopParams lps{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0, opt.ca, opt.cb};
    if (batch > 1)
      NS_CUDA(cudaMemcpyAsync(djobs, jobs.data(), jobs.size() * sizeof(JobParams), cudaMemcpyHostToDevice, st));
    // batch of one: the kernel stores its result record straight into mapped pinned memory (no copy)
    const bool mapped = (batch == 1 && rg.dstate != nullptr);
    NS_CUDA(launch_small(H, ldh, h_stride, batch > 1 ? djobs : nullptr, jobs[0], lps, R, ldr, r_stride,
                         mapped ? rg.dstate : state, batch, st));
    states.resize(batch);
    if (mapped) {
      NS_CUDA(cudaStreamSynchronize(st));
      std::atomic_thread_fence(std::memory_order_acquire);
      std::memcpy(&states[0], rg.pstate, sizeof(DevState));   // written by the kernel
    } else {
      NS_CUDA(cudaMemcpyAsync(states.data(), state, sizeof(DevState) * batch, cudaMemcpyDeviceToHost, st));
      NS_CUDA(cudaStreamSynchronize(st));
    }
    if (launches) *launches = 1;
    return NS_OK;
  }
  NS_CUDA(cudaMemcpyAsync(djobs, jobs.data(), jobs.size() * sizeof(JobParams), cudaMemcpyHostToDevice, st));
  const bool t64 = use_tile64(L.d_pad, batch);
  const int tile_rows = t64 ? k64Tile : kTile;
  const int nb = L.d_pad / tile_rows;                 // tile blocks per dimension (= diagonal partials)
  std::vector<int2> tl = make_tiles(nb);
  const int n_t = (int)tl.size();
  NS_CUDA(cudaMemcpyAsync(tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  // batched: CTA rows follow the compacted active-job list; the grid covers a host-side upper bound of
  // its length (the newest completed n_active readback: the count only decreases)
  int* jlist = reinterpret_cast<int*>(ws + L.off_jlist);
  const bool compact = batch > 1;
  int rows = batch;
  auto product = [&](const CUtensorMap& a, const CUtensorMap& b, ProdParams pp) {
    if (compact && rows < batch) {   // while every job may be active, rows map 1:1 (no list indirection)
      pp.job_list = jlist;
      pp.n_job_list = jlist + batch;
    }
    const int gy = std::max(rows, 1);
    return t64 ? launch_product64(a, b, pp, gy, st) : launch_product(a, b, pp, gy, st);
  };

  CUtensorMap tmA, tmB, tmY;
  ns_status_t s;
  if ((s = encode_map(&tmA, Xa, L.d_pad, batch, tile_rows)) != NS_OK) return s;
  if ((s = encode_map(&tmB, Xb, L.d_pad, batch, tile_rows)) != NS_OK) return s;
  if ((s = encode_map(&tmY, Y, L.d_pad, batch, tile_rows)) != NS_OK) return s;

  NS_CUDA(launch_zero_state(state, batch, n_active, st));
  if (compact) NS_CUDA(launch_compact(state, batch, jlist, jlist + batch, st));
  int nl = compact ? 4 : 3;
  // Host entry (H on the host): H is staged in row chunks into X_b's buffer (dead until update 0) on the
  // side stream; chunk c's rows of X_0 are formed as soon as it lands, and the tiles of the first square
  // whose rows and columns all lie in chunks <= c are launched right after (each CTA writes its partial
  // to the tile's slot of the full list: the decide's sum is unchanged), so the transfer of H overlaps
  // the first product instead of preceding it.
  const bool chunked = opt.h_host != nullptr;   // the host entry checked batch == 1 and the side stream
  const Layout* Lp = &L;
  ProdParams sq0{tiles, n_t, L.d_pad / kBK, L.d, L.d_pad, (long long)L.d_pad * L.d_pad, Y, nullptr, res, state, 0};
  sq0.same_pq = 1;
  if (chunked) {
    SpecCtx& c = spec_ctx();
    const int nch = std::min(8, nb);
    std::vector<int> cb(nch + 1);                   // chunk c = tile blocks [cb[c], cb[c+1])
    for (int q = 0; q <= nch; ++q) cb[q] = (int)((long long)q * nb / nch);
    std::vector<int> chunk_of(nb);
    for (int q = 0; q < nch; ++q)
      for (int b = cb[q]; b < cb[q + 1]; ++b) chunk_of[b] = q;
    std::vector<int2> perm;
    std::vector<int> slot, gstart(nch + 1, 0);
    for (int q = 0; q < nch; ++q) {
      gstart[q] = (int)perm.size();
      for (int t = 0; t < n_t; ++t)
        if (chunk_of[std::max(tl[t].x, tl[t].y)] == q) {
          perm.push_back(tl[t]);
          slot.push_back(t);
        }
    }
    gstart[nch] = (int)perm.size();
    int2* dperm = reinterpret_cast<int2*>(ws + Lp->off_tperm);
    int* dslot = reinterpret_cast<int*>(ws + Lp->off_tslot);
    NS_CUDA(cudaMemcpyAsync(dperm, perm.data(), perm.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    NS_CUDA(cudaMemcpyAsync(dslot, slot.data(), slot.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    NS_CUDA(cudaEventRecord(c.upd, st));             // side stream: X_b is free once the previous call is done
    NS_CUDA(cudaStreamWaitEvent(c.side, c.upd, 0));
    for (int q = 0; q < nch; ++q) {
      const int r0 = cb[q] * tile_rows, r1 = std::min(L.d, cb[q + 1] * tile_rows);
      if (r1 > r0)
        NS_CUDA(cudaMemcpy2DAsync(Xb + (size_t)r0 * L.d_pad, (size_t)L.d_pad * 8, opt.h_host + (size_t)r0 * opt.h_ldh,
                                  (size_t)opt.h_ldh * 8, (size_t)L.d * 8, (size_t)(r1 - r0), cudaMemcpyHostToDevice,
                                  c.side));
      NS_CUDA(cudaEventRecord(c.chunk[q], c.side));
    }
    CUtensorMap tA0;
    ns_status_t s0 = encode_map(&tA0, Xa, L.d_pad, 1, tile_rows);
    if (s0 != NS_OK) return s0;
    for (int q = 0; q < nch; ++q) {
      NS_CUDA(cudaStreamWaitEvent(st, c.chunk[q], 0));
      NS_CUDA(launch_init(Xb, L.d_pad, 0, Xa, djobs, L.d, L.d_pad, 1, st, cb[q] * tile_rows / 64,
                          cb[q + 1] * tile_rows / 64));
      nl += 1;
      if (q == nch - 1) {
        if (t64) NS_CUDA(cudaMemsetAsync(trp, 0, sizeof(double) * nb, st));
        NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, 1, trp, st, nb));
      }
      // groups of the first half of the chunks run while the rest of H is in flight; the tiles of the
      // later chunks go out as one launch once H is complete (separate launches per chunk would each
      // end in a partial wave)
      const int g0 = (q < nch / 2) ? q : nch / 2, g1 = (q < nch / 2) ? q + 1 : nch;
      if ((q < nch / 2 || q == nch - 1) && gstart[g1] > gstart[g0]) {
        ProdParams g = sq0;
        g.tiles = dperm + gstart[g0];
        g.n_tiles = gstart[g1] - gstart[g0];
        g.part_slot = dslot + gstart[g0];
        NS_CUDA(t64 ? launch_product64(tA0, tA0, g, 1, st) : launch_product(tA0, tA0, g, 1, st));
        nl += 1;
      }
    }
  } else {
    NS_CUDA(launch_init(H, ldh, h_stride, Xa, djobs, L.d, L.d_pad, batch, st));
    if (t64) NS_CUDA(cudaMemsetAsync(trp, 0, sizeof(double) * nb * batch, st));
    NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, batch, trp, st, nb));   // 128-block sums, stride nb
  }
  Profiler& pf = prof();
  // event slots: 4 per step (square begin/end, update begin/end)

  LoopParams lp{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0};
  const long long job_stride = (long long)L.d_pad * L.d_pad;
  // Speculative result copy (host entry, one problem): after update j a side-stream kernel copies
  // X_{j+1} to the caller's pinned R if the decide of step j predicted it final (DevState.spec), so the
  // PCIe transfer of the result hides behind the square product that confirms it.  Update j + 2 (which
  // overwrites X_{j+1}'s buffer) waits for that copy.
  SpecCtx* sc = nullptr;
  if (opt.spec_R != nullptr && opt.spec_hit != nullptr && batch == 1 && L.d % 2 == 0 && opt.spec_ldr % 2 == 0 &&
      (reinterpret_cast<uintptr_t>(opt.spec_R) & 15) == 0) {
    SpecCtx& c = spec_ctx();
    if (c.ok) sc = &c;
  }
  int spec_last = 0;                 // largest jn whose copy kernel was enqueued
  // look-ahead: how many steps may be in flight before the host checks the counter
  const double step_flops = 2.0 * (double)L.n_tiles * kTile * kTile * (double)L.d_pad * batch;
  const int LA = opt.lookahead > 0 ? std::min(opt.lookahead, 15) : (step_flops > 2e10 ? 2 : 8);

  for (int j = 0; j <= max_steps; ++j) {
    if (j >= LA) {
      const int slot = (j - LA) % 16;
      NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
      if (rg.slots[slot] == 0) break;
      rows = std::min(rows, rg.slots[slot]);
      if (compact)   // a newer readback may already be in: tighter bound, no wait
        for (int q = j - 1; q > j - LA; --q)
          if (cudaEventQuery(rg.ev[q % 16]) == cudaSuccess) {
            rows = std::min(rows, rg.slots[q % 16]);
            break;
          }
    }
    const bool odd = (j & 1) != 0;
    double* Xc = odd ? Xb : Xa;
    double* Xn = odd ? Xa : Xb;
    const CUtensorMap& tmC = odd ? tmB : tmA;

    ProdParams sq{tiles, n_t, L.d_pad / kBK, L.d, L.d_pad, job_stride, Y, nullptr, res, state, 0};
    sq.same_pq = 1;
    if (pf.on) NS_CUDA(cudaEventRecord(pf.get(4 * j + 0), st));
    if (!(chunked && j == 0)) NS_CUDA(product(tmC, tmC, sq));   // chunked: the first square already ran
    if (pf.on) NS_CUDA(cudaEventRecord(pf.get(4 * j + 1), st));
    NS_CUDA(launch_decide(state, djobs, res, n_t, trp, nb, lp, batch, n_active, st));
    nl += (chunked && j == 0) ? 1 : 2;
    if (compact) {
      NS_CUDA(launch_compact(state, batch, jlist, jlist + batch, st));
      nl += 1;
    }
    if (j < max_steps) {
      ProdParams up{tiles, n_t, L.d_pad / kBK, L.d, L.d_pad, job_stride, Xn, Xc, trp, state, 1, opt.ca, opt.cb};
      if (sc && j >= 2) NS_CUDA(cudaStreamWaitEvent(st, sc->cp[(j - 1) & 1], 0));   // copy of X_{j-1} done
      if (pf.on) NS_CUDA(cudaEventRecord(pf.get(4 * j + 2), st));
      NS_CUDA(product(tmC, tmY, up));
      if (pf.on) NS_CUDA(cudaEventRecord(pf.get(4 * j + 3), st));
      nl += 1;
      if (sc) {
        NS_CUDA(cudaEventRecord(sc->upd, st));
        NS_CUDA(cudaStreamWaitEvent(sc->side, sc->upd, 0));
        NS_CUDA(launch_spec_copy(state, j + 1, Xn, L.d, L.d_pad, opt.spec_R, opt.spec_ldr, sc->side));
        NS_CUDA(cudaEventRecord(sc->cp[(j + 1) & 1], sc->side));
        spec_last = j + 1;
        nl += 1;
      }
    }
    const int slot = j % 16;
    NS_CUDA(cudaMemcpyAsync(&rg.slots[slot], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    NS_CUDA(cudaEventRecord(rg.ev[slot], st));
  }
  NS_CUDA(launch_copy_out(Xa, Xb, L.d, L.d_pad, state, R, ldr, r_stride, batch, st));
  nl += 1;
  if (sc) {
    NS_CUDA(cudaEventRecord(sc->end, sc->side));
    NS_CUDA(cudaStreamWaitEvent(st, sc->end, 0));
  }
  states.resize(batch);
  NS_CUDA(cudaMemcpyAsync(states.data(), state, sizeof(DevState) * batch, cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  if (sc)   // R already holds X_{j} iff the copy kernel for jn = j ran (spec == j at the end)
    *opt.spec_hit = states[0].done && states[0].j >= 1 && states[0].spec == states[0].j && states[0].j <= spec_last;
  if (launches) *launches = nl;
  if (pf.on) {
    // launches that did work: squares j = 0..max_j, updates j = 0..max_j-1 (max over jobs)
    int max_j = 0;
    for (const DevState& d : states) max_j = std::max(max_j, d.j);
    for (int j = 0; j <= max_j; ++j) {
      float ms = 0.f;
      NS_CUDA(cudaEventElapsedTime(&ms, pf.get(4 * j + 0), pf.get(4 * j + 1)));
      pf.acc.ms_square += ms;
      pf.acc.n_square += 1;
      if (j < max_j) {
        NS_CUDA(cudaEventElapsedTime(&ms, pf.get(4 * j + 2), pf.get(4 * j + 3)));
        pf.acc.ms_update += ms;
        pf.acc.n_update += 1;
      }
    }
    pf.acc.n_calls += 1;
  }
  return NS_OK;
}

// An Ozaki product launch (all its K segments), timed for the executed-INT8 roofline when profiling.
cudaError_t oz_product(const CUtensorMap& ta, const CUtensorMap& tb, const OzParams& p, int batch, cudaStream_t st) {
  const int pairs = p.groups >= 8 ? 34 : 28;
  const double work = (double)pairs * 2.0 * kTile * (use_oz_mc() ? kTile : 64) * (double)p.ld * p.n_tiles * batch;
  return xtimed(st, p.mode == 2 ? 3 : 2, work, [&] { return launch_ozaki_product(ta, tb, p, batch, st); });
}

// Ozaki path (single problem): the FP64 loop with every product on the INT8 tensor cores.
// Ozaki path: L.batch problems (H + b*h_stride, R + b*r_stride), every product on the INT8 tensor cores.
// Digit-pair groups for an Ozaki run: 8 when the stopping tolerance is within reach of the 7-group
// residual floor (~1.5e-15 d, absolute), 7 otherwise (21% fewer MACs); NS_OZ_GROUPS=7|8 forces one.
int oz_groups(double tol, ns_tolmode_t tm, int d) {
  static const int forced = [] {
    const char* e = getenv("NS_OZ_GROUPS");
    return e ? atoi(e) : 0;
  }();
  if (forced == 7 || forced == 8) return forced;
  const double tol_abs = (tm == NS_TOL_PER_SQRT_D) ? tol * std::sqrt((double)d) : tol;
  return (tol > 0.0 && tol_abs < 1e-13 * d) ? 8 : 7;
}

ns_status_t run_ozaki_batch(const Layout& L, uint8_t* ws, const double* H, long long ldh, long long h_stride,
                            const std::vector<JobParams>& jobs, int32_t max_steps, double tol, ns_tolmode_t tm,
                            double* R, long long ldr, long long r_stride, cudaStream_t st, const Opts& opt,
                            std::vector<DevState>& states, int* launches) {
  const int batch = (int)L.batch;
  double* Xa = reinterpret_cast<double*>(ws + L.off_xa);
  double* Xb = reinterpret_cast<double*>(ws + L.off_xb);
  double* Y = reinterpret_cast<double*>(ws + L.off_y);
  double* res = reinterpret_cast<double*>(ws + L.off_ores);
  double* trp = reinterpret_cast<double*>(ws + L.off_otr);
  int8_t* slX = reinterpret_cast<int8_t*>(ws + L.off_ozx);
  int8_t* slY = reinterpret_cast<int8_t*>(ws + L.off_ozy);
  int* eX = reinterpret_cast<int*>(ws + L.off_oex);
  int* eY = reinterpret_cast<int*>(ws + L.off_oey);
  int2* otiles = reinterpret_cast<int2*>(ws + L.off_otiles);
  JobParams* djobs = reinterpret_cast<JobParams*>(ws + L.off_jobs);
  DevState* state = reinterpret_cast<DevState*>(ws + L.off_state);
  int* n_active = reinterpret_cast<int*>(ws + L.off_active);
  HostRing& rg = ring();
  if (!rg.ok) return fail(NS_ERR_CUDA, "pinned status ring allocation failed");
  std::vector<int2> ot = oz_tile_list(L.n, true);
  const int nt = (int)ot.size(), npart = oz_partials(ot), ndiag = 2 * L.n;
  const long long js = (long long)L.d_pad * L.d_pad;
  NS_CUDA(cudaMemcpyAsync(otiles, ot.data(), ot.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  NS_CUDA(cudaMemcpyAsync(djobs, jobs.data(), jobs.size() * sizeof(JobParams), cudaMemcpyHostToDevice, st));
  CUtensorMap tXa, tXb, tY;
  ns_status_t s;
  if ((s = encode_map_i8(&tXa, slX, L.d_pad, kOzSlices * batch, kTile)) != NS_OK) return s;
  if ((s = encode_map_i8(&tXb, slX, L.d_pad, kOzSlices * batch, 64)) != NS_OK) return s;
  if ((s = encode_map_i8(&tY, slY, L.d_pad, kOzSlices * batch, 64)) != NS_OK) return s;
  int nl = 0;
  NS_CUDA(launch_zero_state(state, batch, n_active, st));
  NS_CUDA(launch_init(H, ldh, h_stride, Xa, djobs, L.d, L.d_pad, batch, st));
  NS_CUDA(cudaMemsetAsync(trp, 0, sizeof(double) * ndiag * batch, st));
  NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, batch, trp, st, ndiag));
  nl += 3;
  LoopParams lp{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0};
  const int LA = opt.lookahead > 0 ? std::min(opt.lookahead, 15) : (batch > 1 ? 8 : 2);
  for (int j = 0; j <= max_steps; ++j) {
    if (j >= LA) {
      const int slot = (j - LA) % 16;
      NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
      if (rg.slots[slot] == 0) break;
    }
    const bool odd = (j & 1) != 0;
    double* Xc = odd ? Xb : Xa;
    double* Xn = odd ? Xa : Xb;
    NS_CUDA(launch_ozaki_slice(Xc, slX, eX, L.d_pad, batch, st));
    OzParams sq{otiles, nt, L.d_pad / 64, L.d, L.d_pad, js, Y, nullptr, eX, eX, res, state, 0};
    sq.groups = oz_groups(tol, tm, L.d);
    NS_CUDA(oz_product(tXa, tXb, sq, batch, st));
    NS_CUDA(launch_decide(state, djobs, res, npart, trp, ndiag, lp, batch, n_active, st));
    nl += 3;
    if (j < max_steps) {
      NS_CUDA(launch_ozaki_slice(Y, slY, eY, L.d_pad, batch, st));
      OzParams up{otiles, nt, L.d_pad / 64, L.d, L.d_pad, js, Xn, Xc, eX, eY, trp, state, 1, opt.ca, opt.cb};
      up.groups = sq.groups;
      NS_CUDA(oz_product(tXa, tY, up, batch, st));
      nl += 2;
    }
    NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
  }
  NS_CUDA(launch_copy_out(Xa, Xb, L.d, L.d_pad, state, R, ldr, r_stride, batch, st));
  nl += 1;
  states.resize(batch);
  NS_CUDA(cudaMemcpyAsync(states.data(), state, sizeof(DevState) * batch, cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  if (launches) *launches = nl;
  return NS_OK;
}

ns_status_t run_ozaki(const Layout& L, uint8_t* ws, const double* H, long long ldh, const JobParams& jp,
                      int32_t max_steps, double tol, ns_tolmode_t tm, double* R, long long ldr, cudaStream_t st,
                      const Opts& opt, DevState& out_state, int* launches) {
  std::vector<DevState> states;
  const ns_status_t s = run_ozaki_batch(L, ws, H, ldh, 0, std::vector<JobParams>{jp}, max_steps, tol, tm, R, ldr, 0,
                                        st, opt, states, launches);
  if (s == NS_OK) out_state = states[0];
  return s;
}

// General odd sign-preserving polynomial filter steps (eq:signpreserving P:278-289, the
// "low-degree odd polynomial filters" of P:513-518): X_{j+1} = phi(X_j) = sum_{i=0}^{m} c_i X_j^{2i+1}
// = X_j P(Y_j), P(y) = sum_i c_i y^i, Y_j = X_j^2, degree m >= 2 in Y (m = 1 is the cubic step of run_loop).
// P(Y) is formed by Horner's rule in Y with symmetric products (every Horner iterate is a polynomial in Y,
// so it commutes with Y and X and the upper-tile products with mirrored writes apply):
//   T_{m-2} = c_m Y Y + c_{m-1} Y + c_{m-2} I         (product Y.Y; mode-1 epilogue ca = c_{m-1}, cb = c_m, cc)
//   T_i     = T_{i+1} Y + c_i I,  i = m-3 .. 0          (mode 1, ca = 0, cb = 1, cc = c_i)
//   X_{j+1} = X_j T_0                                   (mode 1, ca = 0, cb = 1: trace partials of X_{j+1})
// m + 1 products per step (the square + m - 1 Horner + 1), one extra d_pad^2 buffer E (T_i in E for even i,
// in X_{j+1}'s buffer for odd i).  The square, residual, decide and stop rule are the NS loop's.  FP64 DMMA
// or the Ozaki INT8 products (the operands of every product are re-sliced as needed).
ns_status_t run_filter(const Layout& L, uint8_t* ws, const double* H, long long ldh, const JobParams& jp,
                       int32_t max_steps, double tol, ns_tolmode_t tm, double* R, long long ldr, cudaStream_t st,
                       const Opts& opt, bool ozaki, DevState& out_state, int* launches) {
  double c[kMaxFilterDeg + 1] = {opt.ca, opt.cb};
  for (int i = 2; i <= kMaxFilterDeg; ++i) c[i] = opt.cz[i - 2];
  int m = kMaxFilterDeg;
  while (m > 2 && c[m] == 0.0) --m;
  double* Xa = reinterpret_cast<double*>(ws + L.off_xa);
  double* Xb = reinterpret_cast<double*>(ws + L.off_xb);
  double* Y = reinterpret_cast<double*>(ws + L.off_y);
  double* E = reinterpret_cast<double*>(ws + align256(L.total));
  JobParams* djobs = reinterpret_cast<JobParams*>(ws + L.off_jobs);
  DevState* state = reinterpret_cast<DevState*>(ws + L.off_state);
  int* n_active = reinterpret_cast<int*>(ws + L.off_active);
  HostRing& rg = ring();
  if (!rg.ok) return fail(NS_ERR_CUDA, "pinned status ring allocation failed");
  NS_CUDA(cudaMemcpyAsync(djobs, &jp, sizeof(JobParams), cudaMemcpyHostToDevice, st));
  ns_status_t s;
  int nl = 0;
  LoopParams lp{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0};
  const int LA = opt.lookahead > 0 ? std::min(opt.lookahead, 15) : 2;
  NS_CUDA(launch_zero_state(state, 1, n_active, st));
  NS_CUDA(launch_init(H, ldh, 0, Xa, djobs, L.d, L.d_pad, 1, st));
  nl += 2;
  if (!ozaki) {
    double* res = reinterpret_cast<double*>(ws + L.off_res);
    double* trp = reinterpret_cast<double*>(ws + L.off_tr);
    int2* tiles = reinterpret_cast<int2*>(ws + L.off_tiles);
    const bool t64 = use_tile64(L.d_pad, 1);
    const int tile_rows = t64 ? k64Tile : kTile;
    const int nb = L.d_pad / tile_rows;
    const std::vector<int2> tl = make_tiles(nb);
    const int n_t = (int)tl.size();
    NS_CUDA(cudaMemcpyAsync(tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    CUtensorMap tmA, tmB, tmY, tmE;
    if ((s = encode_map(&tmA, Xa, L.d_pad, 1, tile_rows)) != NS_OK) return s;
    if ((s = encode_map(&tmB, Xb, L.d_pad, 1, tile_rows)) != NS_OK) return s;
    if ((s = encode_map(&tmY, Y, L.d_pad, 1, tile_rows)) != NS_OK) return s;
    if ((s = encode_map(&tmE, E, L.d_pad, 1, tile_rows)) != NS_OK) return s;
    auto product = [&](const CUtensorMap& a, const CUtensorMap& b, const ProdParams& pp) {
      ++nl;
      return t64 ? launch_product64(a, b, pp, 1, st) : launch_product(a, b, pp, 1, st);
    };
    if (t64) NS_CUDA(cudaMemsetAsync(trp, 0, sizeof(double) * nb, st));
    NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, 1, trp, st, nb));
    ++nl;
    for (int j = 0; j <= max_steps; ++j) {
      if (j >= LA) {
        const int slot = (j - LA) % 16;
        NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
        if (rg.slots[slot] == 0) break;
      }
      const bool odd = (j & 1) != 0;
      double* Xc = odd ? Xb : Xa;
      double* Xn = odd ? Xa : Xb;
      const CUtensorMap& tC = odd ? tmB : tmA;
      const CUtensorMap& tN = odd ? tmA : tmB;
      ProdParams sq{tiles, n_t, L.d_pad / kBK, L.d, L.d_pad, 0, Y, nullptr, res, state, 0};
      NS_CUDA(product(tC, tC, sq));
      NS_CUDA(launch_decide(state, djobs, res, n_t, trp, nb, lp, 1, n_active, st));
      ++nl;
      if (j < max_steps) {
        for (int i = m - 2; i >= 0; --i) {     // Horner in Y; the partial buffer res is free after the decide
          const bool first = (i == m - 2);
          double* A = first ? Y : (((i + 1) % 2 == 0) ? E : Xn);
          const CUtensorMap& tAm = first ? tmY : (((i + 1) % 2 == 0) ? tmE : tN);
          double* T = (i % 2 == 0) ? E : Xn;
          ProdParams hp{tiles, n_t, L.d_pad / kBK, L.d, L.d_pad, 0, T, A, res, state, 1,
                        first ? c[m - 1] : 0.0, first ? c[m] : 1.0};
          hp.cc = c[i];
          NS_CUDA(product(tAm, tmY, hp));
        }
        ProdParams fp{tiles, n_t, L.d_pad / kBK, L.d, L.d_pad, 0, Xn, Xc, trp, state, 1, 0.0, 1.0};
        NS_CUDA(product(tC, tmE, fp));
      }
      NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
    }
  } else {
    double* res = reinterpret_cast<double*>(ws + L.off_ores);
    double* trp = reinterpret_cast<double*>(ws + L.off_otr);
    int8_t* slX = reinterpret_cast<int8_t*>(ws + L.off_ozx);
    int8_t* slY = reinterpret_cast<int8_t*>(ws + L.off_ozy);
    int* eX = reinterpret_cast<int*>(ws + L.off_oex);
    int* eY = reinterpret_cast<int*>(ws + L.off_oey);
    int2* otiles = reinterpret_cast<int2*>(ws + L.off_otiles);
    const std::vector<int2> ot = oz_tile_list(L.n, true);
    const int nt = (int)ot.size(), npart = oz_partials(ot), ndiag = 2 * L.n;
    NS_CUDA(cudaMemcpyAsync(otiles, ot.data(), ot.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    CUtensorMap tXa, tXb, tYa, tY;
    if ((s = encode_map_i8(&tXa, slX, L.d_pad, kOzSlices, kTile)) != NS_OK) return s;
    if ((s = encode_map_i8(&tXb, slX, L.d_pad, kOzSlices, 64)) != NS_OK) return s;
    if ((s = encode_map_i8(&tYa, slY, L.d_pad, kOzSlices, kTile)) != NS_OK) return s;
    if ((s = encode_map_i8(&tY, slY, L.d_pad, kOzSlices, 64)) != NS_OK) return s;
    const int groups = oz_groups(tol, tm, L.d);
    NS_CUDA(cudaMemsetAsync(trp, 0, sizeof(double) * ndiag, st));
    NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, 1, trp, st, ndiag));
    ++nl;
    for (int j = 0; j <= max_steps; ++j) {
      if (j >= LA) {
        const int slot = (j - LA) % 16;
        NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
        if (rg.slots[slot] == 0) break;
      }
      const bool odd = (j & 1) != 0;
      double* Xc = odd ? Xb : Xa;
      double* Xn = odd ? Xa : Xb;
      NS_CUDA(launch_ozaki_slice(Xc, slX, eX, L.d_pad, 1, st));
      OzParams sq{otiles, nt, L.d_pad / 64, L.d, L.d_pad, 0, Y, nullptr, eX, eX, res, state, 0};
      sq.groups = groups;
      NS_CUDA(oz_product(tXa, tXb, sq, 1, st));
      NS_CUDA(launch_decide(state, djobs, res, npart, trp, ndiag, lp, 1, n_active, st));
      nl += 3;
      if (j < max_steps) {
        NS_CUDA(launch_ozaki_slice(Y, slY, eY, L.d_pad, 1, st));
        ++nl;
        for (int i = m - 2; i >= 0; --i) {
          const bool first = (i == m - 2);
          double* A = first ? Y : (((i + 1) % 2 == 0) ? E : Xn);
          if (!first) {                        // A-operand digits of T_{i+1} (X_j's digits are re-sliced below)
            NS_CUDA(launch_ozaki_slice(A, slX, eX, L.d_pad, 1, st));
            ++nl;
          }
          double* T = (i % 2 == 0) ? E : Xn;
          OzParams hp{otiles, nt, L.d_pad / 64, L.d, L.d_pad, 0, T, A, first ? eY : eX, eY, res, state, 1,
                      first ? c[m - 1] : 0.0, first ? c[m] : 1.0};
          hp.cc = c[i];
          hp.groups = groups;
          NS_CUDA(oz_product(first ? tYa : tXa, tY, hp, 1, st));
          ++nl;
        }
        if (m >= 3) {
          NS_CUDA(launch_ozaki_slice(Xc, slX, eX, L.d_pad, 1, st));
          ++nl;
        }
        NS_CUDA(launch_ozaki_slice(E, slY, eY, L.d_pad, 1, st));   // T_0 (Y's digits are no longer needed)
        OzParams fp{otiles, nt, L.d_pad / 64, L.d, L.d_pad, 0, Xn, Xc, eX, eY, trp, state, 1, 0.0, 1.0};
        fp.groups = groups;
        NS_CUDA(oz_product(tXa, tY, fp, 1, st));
        nl += 2;
      }
      NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
    }
  }
  NS_CUDA(launch_copy_out(Xa, Xb, L.d, L.d_pad, state, R, ldr, 0, 1, st));
  ++nl;
  NS_CUDA(cudaMemcpyAsync(&out_state, state, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  if (launches) *launches = nl;
  return NS_OK;
}

// Mixed path (single problem): BF16x3 tcgen05 steps -> switch -> re-anchor -> FP64 steps.
ns_status_t run_mixed(const Layout& L, uint8_t* ws, const double* H, long long ldh, const JobParams& jp,
                      int32_t max_steps, double tol, ns_tolmode_t tm, double* R, long long ldr, cudaStream_t st,
                      const Opts& opt, DevState& out_state, int* launches, bool tf32 = false) {
  const int mx_nkb = L.d_pad / (tf32 ? 32 : kMxBK);
  double* Xa = reinterpret_cast<double*>(ws + L.off_xa);
  double* Xb = reinterpret_cast<double*>(ws + L.off_xb);
  double* Y = reinterpret_cast<double*>(ws + L.off_y);
  double* Ahat = reinterpret_cast<double*>(ws + L.off_ahat);
  double* Rc = reinterpret_cast<double*>(ws + L.off_r);
  double* Pc = reinterpret_cast<double*>(ws + L.off_p);
  double* res = reinterpret_cast<double*>(ws + L.off_res);
  double* trp = reinterpret_cast<double*>(ws + L.off_tr);
  double* cgpart = reinterpret_cast<double*>(ws + L.off_cgpart);
  CgScalars* cgsc = reinterpret_cast<CgScalars*>(ws + L.off_cgsc);
  void* PXa = ws + L.off_px;
  void* PXb = ws + L.off_pxb;
  void* PY = ws + L.off_py;
  int2* tiles = reinterpret_cast<int2*>(ws + L.off_tiles);
  int2* full = reinterpret_cast<int2*>(ws + L.off_full);
  JobParams* djobs = reinterpret_cast<JobParams*>(ws + L.off_jobs);
  DevState* state = reinterpret_cast<DevState*>(ws + L.off_state);
  int* n_active = reinterpret_cast<int*>(ws + L.off_active);
  HostRing& rg = ring();
  if (!rg.ok) return fail(NS_ERR_CUDA, "pinned status ring allocation failed");
  const size_t mat_bytes = (size_t)L.d_pad * L.d_pad * sizeof(double);

  std::vector<int2> tl = make_tiles(L.n), tf = make_tiles_full(L.n);
  NS_CUDA(cudaMemcpyAsync(tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  NS_CUDA(cudaMemcpyAsync(full, tf.data(), tf.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  NS_CUDA(cudaMemcpyAsync(djobs, &jp, sizeof(JobParams), cudaMemcpyHostToDevice, st));
  // split-precision products: 2-SM kernel on 256 x 128 pair tiles (BF16x3 default: 2.08 vs 2.10 s at cfg3)
  // or the one-SM kernel (TF32x3: 2.92 s vs 3.01 s with the pair kernel)
  const bool mx2 = use_mx2() && !tf32;
  int2* ptiles = reinterpret_cast<int2*>(ws + L.off_ptiles);
  int2* pfull = reinterpret_cast<int2*>(ws + L.off_pfull);
  const std::vector<int2> ps = mx2 ? make_tiles_pairs(L.n, true) : std::vector<int2>();
  const std::vector<int2> pf = mx2 ? make_tiles_pairs(L.n, false) : std::vector<int2>();
  if (mx2) {
    NS_CUDA(cudaMemcpyAsync(ptiles, ps.data(), ps.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    NS_CUDA(cudaMemcpyAsync(pfull, pf.data(), pf.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  }
  const int2* mx_sym = mx2 ? ptiles : tiles;
  const int2* mx_full = mx2 ? pfull : full;
  const int mx_nsym = mx2 ? 2 * (int)ps.size() : L.n_tiles;     // CTAs (= residual partials) per product
  const int mx_nfull = mx2 ? 2 * (int)pf.size() : L.n * L.n;

  CUtensorMap tmA, tmB, tmY, tmAh, tmPXa, tmPXb, tmPY, tqPXa, tqPXb, tqPY;   // tq*: Q-operand maps
  ns_status_t s;
  if ((s = encode_map(&tmA, Xa, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map(&tmB, Xb, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map(&tmY, Y, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map(&tmAh, Ahat, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map_bf16(&tmPXa, PXa, L.d_pad, 2, tf32)) != NS_OK) return s;
  if ((s = encode_map_bf16(&tmPXb, PXb, L.d_pad, 2, tf32)) != NS_OK) return s;
  if ((s = encode_map_bf16(&tmPY, PY, L.d_pad, 2, tf32)) != NS_OK) return s;
  const int qrows = mx2 ? 64 : kTile;
  if ((s = encode_map_bf16(&tqPXa, PXa, L.d_pad, 2, tf32, qrows)) != NS_OK) return s;
  if ((s = encode_map_bf16(&tqPXb, PXb, L.d_pad, 2, tf32, qrows)) != NS_OK) return s;
  if ((s = encode_map_bf16(&tqPY, PY, L.d_pad, 2, tf32, qrows)) != NS_OK) return s;
  auto mx_product = [&](const CUtensorMap& tP, const CUtensorMap& tQ, const MxParams& mp) {
    // executed low-precision flops: 3 GEMMs (hi*hi, hi*lo, lo*hi) on every 128x128 output tile computed
    const double work = tf32 ? 0.0 : 3.0 * 2.0 * kTile * kTile * (double)L.d_pad * mp.n_tiles;
    return xtimed(st, mp.mode == 2 ? 1 : 0, work, [&] {
      return mx2 ? launch_mx2_product(tP, tQ, mp, 1, st) : launch_mx_product(tP, tQ, mp, 1, st);
    });
  };

  int nl = 0;
  NS_CUDA(launch_zero_state(state, 1, n_active, st));
  NS_CUDA(launch_init(H, ldh, 0, Xa, djobs, L.d, L.d_pad, 1, st));
  NS_CUDA(cudaMemcpyAsync(Ahat, Xa, mat_bytes, cudaMemcpyDeviceToDevice, st));
  NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, 1, trp, st));
  NS_CUDA(launch_split_planes(Xa, PXa, L.d_pad, 1, st, tf32));
  nl += 4;

  // ---------------- phase 1: BF16x3 steps until the switch threshold ----------------
  // run-to-tolerance: switch at the first r_j/sqrt(d) < switch_tol (C16).  Fixed-step mode (tol = 0):
  // low precision up to j = max_steps - kPolishSteps, then re-anchor and kPolishSteps FP64 steps.
  const int kPolishSteps = 2;
  const int switch_at = (tol == 0.0) ? std::max(0, max_steps - kPolishSteps) : -1;
  LoopParams lp_low{L.d, L.d_pad, max_steps, (int)tm, tol, opt.switch_tol > 0 ? opt.switch_tol : 1e-300, switch_at, 1};
  const int LA = opt.lookahead > 0 ? std::min(opt.lookahead, 15) : 2;
  const long long js = (long long)L.d_pad * L.d_pad;
  for (int j = 0; j <= max_steps; ++j) {
    if (j >= LA) {
      const int slot = (j - LA) % 16;
      NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
      if (rg.slots[slot] == 0) break;
    }
    const bool odd = (j & 1) != 0;
    double* Xc = odd ? Xb : Xa;
    double* Xn = odd ? Xa : Xb;
    const CUtensorMap& tPc = odd ? tmPXb : tmPXa;
    const CUtensorMap& tQc = odd ? tqPXb : tqPXa;
    void* PXn = odd ? PXa : PXb;
    MxParams sq{mx_sym, mx_nsym, mx_nkb, L.d, L.d_pad, js, Y, nullptr, PY, res, state, 0, tf32 ? 1 : 0};
    NS_CUDA(mx_product(tPc, tQc, sq));
    NS_CUDA(launch_decide(state, djobs, res, mx_nsym, trp, L.n, lp_low, 1, n_active, st));
    nl += 2;
    if (j < max_steps) {
      MxParams up{mx_sym, mx_nsym, mx_nkb, L.d, L.d_pad, js, Xn, Xc, PXn, trp, state, 1, tf32 ? 1 : 0};
      NS_CUDA(mx_product(tPc, tqPY, up));
      nl += 1;
    }
    NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
  }
  DevState hs;
  NS_CUDA(cudaMemcpyAsync(&hs, state, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));

  if (!hs.done && !opt.stop_at_switch && hs.sw) {
    const int j0 = hs.j;
    double* Xt = (j0 & 1) ? Xb : Xa;                // X~ = X_switch
    double* Xo = (j0 & 1) ? Xa : Xb;                // free FP64 buffer
    const CUtensorMap& tXt = (j0 & 1) ? tmB : tmA;
    const CUtensorMap& tXo = (j0 & 1) ? tmA : tmB;
    const int nk = L.d_pad / kBK;
    // polish 1: re-anchor products and polishing steps on the Ozaki INT8 products; 2: only the re-anchor's
    // two dense products (the polishing steps stay FP64 DMMA)
    const bool oz = (opt.polish >= 1);
    const bool oz_steps = (opt.polish == 1);
    int8_t* slX = reinterpret_cast<int8_t*>(ws + L.off_ozx);
    int8_t* slY = reinterpret_cast<int8_t*>(ws + L.off_ozy);
    int* eX = reinterpret_cast<int*>(ws + L.off_oex);
    int* eY = reinterpret_cast<int*>(ws + L.off_oey);
    double* ores = reinterpret_cast<double*>(ws + L.off_ores);
    double* otr = reinterpret_cast<double*>(ws + L.off_otr);
    int2* otiles = reinterpret_cast<int2*>(ws + L.off_otiles);
    CUtensorMap tOa, tOb, tOy;
    if (oz) {
      if ((s = encode_map_i8(&tOa, slX, L.d_pad, kOzSlices, kTile)) != NS_OK) return s;
      if ((s = encode_map_i8(&tOb, slX, L.d_pad, kOzSlices, 64)) != NS_OK) return s;
      if ((s = encode_map_i8(&tOy, slY, L.d_pad, kOzSlices, 64)) != NS_OK) return s;
    }
    const std::vector<int2> ot_full = oz ? oz_tile_list(L.n, false) : std::vector<int2>();
    // C = P Q^T over every tile (P, Q row panels), FP64 DMMA or Ozaki
    auto dense = [&](const double* P, const CUtensorMap& tP, const double* Q, const CUtensorMap& tQ,
                     double* C) -> ns_status_t {
      if (oz) {
        NS_CUDA(launch_ozaki_slice(P, slX, eX, L.d_pad, 1, st));
        NS_CUDA(launch_ozaki_slice(Q, slY, eY, L.d_pad, 1, st));
        OzParams pp{otiles, (int)ot_full.size(), L.d_pad / 64, L.d, L.d_pad, 0, C, nullptr, eX, eY, nullptr, nullptr, 2};
        NS_CUDA(oz_product(tOa, tOy, pp, 1, st));
        nl += 3;
      } else {
        ProdParams pp{full, L.n * L.n, nk, L.d, L.d_pad, 0, C, nullptr, nullptr, nullptr, 2};
        NS_CUDA(launch_product(tP, tQ, pp, 1, st));
        nl += 1;
      }
      return NS_OK;
    };
    // Late switch (reading C16b): quadratic convergence can carry the residual from above the switch threshold to
    // below the split-precision noise floor in one step; X_switch then sits as close to its reflector as the
    // low-precision steps' eigenvalue noise, and the FP64 residuals that follow deviate from the exact recurrence's by tens of
    // percent (measured: +-1 step in 4 of 332 random runs).  When the low-precision residual at the switch reads
    // below kRedoFloor (it cannot resolve less), the last low-precision step is taken again in FP64-class arithmetic
    // from X_{j0-1}, which is still in the other buffer (its distance to the reflector is >= the switch threshold,
    // two decades above the noise): X_switch := 1.5 X_{j0-1} - 0.5 X_{j0-1}^3.  Run-to-tolerance mode only (a fixed
    // step count does not depend on residuals).  NS_MIXED_REDO=0 disables (experiments).
    static const bool redo_env = [] {
      const char* e = getenv("NS_MIXED_REDO");
      return !(e && e[0] == '0');
    }();
    constexpr double kRedoFloor = 5e-4;
    if (redo_env && tol > 0.0 && j0 >= 1 && opt.ca == 1.5 && opt.cb == -0.5 &&
        hs.sw_residual < kRedoFloor * std::sqrt((double)L.d)) {
      if (oz) {
        const std::vector<int2> ot = oz_tile_list(L.n, true);
        NS_CUDA(cudaMemcpyAsync(otiles, ot.data(), ot.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
        NS_CUDA(launch_ozaki_slice(Xo, slX, eX, L.d_pad, 1, st));
        OzParams sq{otiles, (int)ot.size(), L.d_pad / 64, L.d, L.d_pad, 0, Y, nullptr, eX, eX, ores, nullptr, 0};
        sq.groups = oz_groups(tol, tm, L.d);
        NS_CUDA(oz_product(tOa, tOb, sq, 1, st));
        NS_CUDA(launch_ozaki_slice(Y, slY, eY, L.d_pad, 1, st));
        OzParams up{otiles, (int)ot.size(), L.d_pad / 64, L.d, L.d_pad, 0, Xt, Xo, eX, eY, otr, nullptr, 1};
        up.groups = sq.groups;
        NS_CUDA(oz_product(tOa, tOy, up, 1, st));
        nl += 4;
      } else {
        ProdParams sq{tiles, L.n_tiles, nk, L.d, L.d_pad, js, Y, nullptr, res, nullptr, 0};
        NS_CUDA(launch_product(tXo, tXo, sq, 1, st));
        ProdParams up{tiles, L.n_tiles, nk, L.d, L.d_pad, js, Xt, Xo, trp, nullptr, 1};
        NS_CUDA(launch_product(tXo, tmY, up, 1, st));
        nl += 2;
      }
    }
    if (oz) NS_CUDA(cudaMemcpyAsync(otiles, ot_full.data(), ot_full.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    // One re-anchor pass: M = A X~, C = M - M^T, F = sym(X~ C) in FP64-class arithmetic, CG on
    // |A|E + E|A| = F with the split-precision operator, X~ <- X~ - E.  Returns the CG iterations used.
    auto reanchor_pass = [&](int* iters) -> ns_status_t {
      // M = A X~  (every tile) -> Y
      if ((s = dense(Ahat, tmAh, Xt, tXt, Y)) != NS_OK) return s;
      // C = M - M^T -> Xo ; |A| = sym(M) -> bf16 planes PY
      NS_CUDA(launch_commutator(Y, Xo, PY, L.d_pad, st, tf32));
      // F' = X~ C^T = -X~ C  (every tile) -> Y
      if ((s = dense(Xt, tXt, Xo, tXo, Y)) != NS_OK) return s;
      // F = sym(X~ C); R = P = F; E = 0 (E overwrites F' in Y tile pair by tile pair; A stays for a
      // second pass)
      int np = 0;
      double* E = Y;
      NS_CUDA(launch_cg_init(Y, Rc, Pc, E, cgpart, L.d_pad, st, &np));
      NS_CUDA(launch_cg_scalar(cgsc, cgpart, np, 0, st, cg_tol() * cg_tol()));
      NS_CUDA(launch_split_planes(Pc, PXa, L.d_pad, 1, st, tf32));
      nl += 4;
      // The host stops enqueuing iterations kCgLag iterations after the device flagged convergence (the
      // flag is read back through the status ring); launches already queued return at once.
      constexpr int kCgLag = 2;
      for (int it = 0; it < opt.cg_iters; ++it) {
        if (it >= kCgLag) {
          const int slot = (it - kCgLag) % 16;
          NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
          if (rg.slots[slot] != 0) break;
        }
        // W = |A| P (BF16x3 tcgen05, every tile) -> Xo
        MxParams pw{mx_full, mx_nfull, mx_nkb, L.d, L.d_pad, 0, Xo, nullptr, nullptr, nullptr, nullptr, 2, tf32 ? 1 : 0};
        pw.skip = &cgsc->done;
        NS_CUDA(mx_product(tmPY, tqPXa, pw));
        NS_CUDA(launch_cg_pw(Pc, Xo, cgpart, L.d_pad, st, cgsc));
        NS_CUDA(launch_cg_scalar(cgsc, cgpart, kEwBlocks, 1, st));
        NS_CUDA(launch_cg_update(E, Rc, Pc, Xo, cgsc, cgpart, L.d_pad, st, &np));
        NS_CUDA(launch_cg_scalar(cgsc, cgpart, np, 2, st));
        nl += 5;
        if (it + 1 < opt.cg_iters) {
          NS_CUDA(launch_cg_direction(Pc, Rc, cgsc, PXa, L.d_pad, st, tf32));
          nl += 1;
        }
        NS_CUDA(cudaMemcpyAsync(&rg.slots[it % 16], &cgsc->done, sizeof(int), cudaMemcpyDeviceToHost, st));
        NS_CUDA(cudaEventRecord(rg.ev[it % 16], st));
      }
      NS_CUDA(launch_apply_correction(Xt, E, L.d_pad, st));
      nl += 1;
      CgScalars h{};
      NS_CUDA(cudaMemcpyAsync(&h, cgsc, sizeof(CgScalars), cudaMemcpyDeviceToHost, st));
      NS_CUDA(cudaStreamSynchronize(st));
      if (getenv("NS_CG_DEBUG"))
        fprintf(stderr, "re-anchor CG: %d iterations, |r|/|r0| = %.3e (tol %.1e, cap %d)\n", h.iters,
                h.rr0 > 0 ? sqrt(h.rr / h.rr0) : 0.0, cg_tol(), opt.cg_iters);
      *iters = h.iters;
      return NS_OK;
    };
    if (opt.cg_iters > 0) {
      // A slowly converging solve means a badly conditioned |A| (small min |x| of X_0): the solution's
      // error from the split-precision operator is amplified by that condition number, so a second pass
      // (iterative refinement: the new right-hand side is formed in FP64 from the corrected iterate)
      // removes what the first left.
      int iters = 0;
      if ((s = reanchor_pass(&iters)) != NS_OK) return s;
      // ... and for d <= kCgRefineMaxD always: there a pass costs a few ms, and the split-precision
      // operator's error floor can reach 1e-10 even at cfg3-like conditioning (randomised stress: d = 278,
      // min|x| = 0.048, 1.3e-10 after one pass, 4e-14 after two)
      const bool ill = iters > kCgRefineIters || hs.j_small >= kCgRefineJSmall || L.d <= kCgRefineMaxD;
      if (ill && (s = reanchor_pass(&iters)) != NS_OK) return s;
    }
    // ---------------- phase 2: FP64-class steps from j0 to tolerance ----------------
    LoopParams lp{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0};
    const int one = 1;
    NS_CUDA(cudaMemcpyAsync(n_active, &one, sizeof(int), cudaMemcpyHostToDevice, st));
    if (oz_steps) {
      // Ozaki steps (as run_ozaki): symmetric 128x64 tile list, its residual / trace partial layouts
      const std::vector<int2> ot = oz_tile_list(L.n, true);
      const int nt = (int)ot.size(), npart = oz_partials(ot), ndiag = 2 * L.n;
      NS_CUDA(cudaMemcpyAsync(otiles, ot.data(), ot.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
      NS_CUDA(cudaMemsetAsync(otr, 0, sizeof(double) * ndiag, st));
      NS_CUDA(launch_trace_partials(Xt, L.d, L.d_pad, 1, otr, st));
      nl += 1;
      for (int j = j0; j <= max_steps; ++j) {
        if (j >= j0 + LA) {
          const int slot = (j - LA) % 16;
          NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
          if (rg.slots[slot] == 0) break;
        }
        const bool odd = (j & 1) != 0;
        double* Xc = odd ? Xb : Xa;
        double* Xn = odd ? Xa : Xb;
        NS_CUDA(launch_ozaki_slice(Xc, slX, eX, L.d_pad, 1, st));
        OzParams sq{otiles, nt, L.d_pad / 64, L.d, L.d_pad, 0, Y, nullptr, eX, eX, ores, state, 0};
        sq.groups = oz_groups(tol, tm, L.d);
        NS_CUDA(oz_product(tOa, tOb, sq, 1, st));
        NS_CUDA(launch_decide(state, djobs, ores, npart, otr, ndiag, lp, 1, n_active, st));
        nl += 3;
        if (j < max_steps) {
          NS_CUDA(launch_ozaki_slice(Y, slY, eY, L.d_pad, 1, st));
          OzParams up{otiles, nt, L.d_pad / 64, L.d, L.d_pad, 0, Xn, Xc, eX, eY, otr, state, 1, opt.ca, opt.cb};
          up.groups = sq.groups;
          NS_CUDA(oz_product(tOa, tOy, up, 1, st));
          nl += 2;
        }
        NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
        NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
      }
    }
    if (!oz_steps) {
    NS_CUDA(launch_trace_partials(Xt, L.d, L.d_pad, 1, trp, st));
    nl += 1;
    for (int j = j0; j <= max_steps; ++j) {
      if (j >= j0 + LA) {
        const int slot = (j - LA) % 16;
        NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
        if (rg.slots[slot] == 0) break;
      }
      const bool odd = (j & 1) != 0;
      double* Xc = odd ? Xb : Xa;
      double* Xn = odd ? Xa : Xb;
      const CUtensorMap& tmC = odd ? tmB : tmA;
      ProdParams sq{tiles, L.n_tiles, nk, L.d, L.d_pad, js, Y, nullptr, res, state, 0};
      NS_CUDA(launch_product(tmC, tmC, sq, 1, st));
      NS_CUDA(launch_decide(state, djobs, res, L.n_tiles, trp, L.n, lp, 1, n_active, st));
      nl += 2;
      if (j < max_steps) {
        ProdParams up{tiles, L.n_tiles, nk, L.d, L.d_pad, js, Xn, Xc, trp, state, 1};
        NS_CUDA(launch_product(tmC, tmY, up, 1, st));
        nl += 1;
      }
      NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
      NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
    }
    }
  }
  NS_CUDA(launch_copy_out(Xa, Xb, L.d, L.d_pad, state, R, ldr, 0, 1, st));
  nl += 1;
  NS_CUDA(cudaMemcpyAsync(&out_state, state, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  if (launches) *launches = nl;
  return NS_OK;
}

// ---------------- sharded (multi-GPU) path ----------------
struct ShardLayout {
  Layout base;
  int nranks = 1, rank = 0, n_my = 0, n_my_max = 0, n_chunks = 1, cs = 0;
  size_t off_my = 0, off_send = 0, off_recv = 0, off_rsend = 0, off_rrecv = 0, off_ptrs = 0, off_ipc = 0, total = 0;
};

ShardLayout make_shard_layout(int64_t d, int nranks, int rank) {
  ShardLayout S;
  S.base = make_layout(d, 1, false);
  S.nranks = nranks;
  S.rank = rank;
  const int nt = S.base.n_tiles;
  S.n_my_max = (nt + nranks - 1) / nranks;
  S.n_my = (nt - rank + nranks - 1) / nranks;   // tiles t = rank, rank + P, ...
  S.n_chunks = std::max(1, std::min(8, S.n_my_max));
  S.cs = (S.n_my_max + S.n_chunks - 1) / S.n_chunks;   // slots per chunk (padded, equal on all ranks)
  size_t o = S.base.total;
  const size_t tile_bytes = (size_t)kTile * kTile * sizeof(double);
  S.off_my = o; o = align256(o + sizeof(int2) * (size_t)S.n_my_max);
  S.off_send = o; o = align256(o + tile_bytes * (size_t)S.n_chunks * S.cs);
  S.off_recv = o; o = align256(o + tile_bytes * (size_t)S.n_chunks * S.cs * (size_t)nranks);
  S.off_rsend = o; o = align256(o + sizeof(double));
  S.off_rrecv = o; o = align256(o + sizeof(double) * (size_t)nranks);
  S.off_ptrs = o; o = align256(o + sizeof(double*) * 6 * (size_t)nranks);   // peer bases: Y, Xa, Xb, res, tr0, tr1
  S.off_ipc = o; o = align256(o + 128 * ((size_t)nranks + 1));              // IPC handle exchange
  S.total = o;
  return S;
}

std::vector<int2> shard_tiles(const std::vector<int2>& all, int nranks, int rank) {
  std::vector<int2> v;
  for (size_t t = (size_t)rank; t < all.size(); t += (size_t)nranks) v.push_back(all[t]);
  return v;
}

#define NS_NCCL(x)                                                                                  \
  do {                                                                                              \
    ncclResult_t r_ = (x);                                                                          \
    if (r_ != ncclSuccess) return fail(NS_ERR_NCCL, "%s failed: %s", #x, ncclGetErrorString(r_)); \
  } while (0)

// Host control plane (ns_comm_init_host): the library's collectives go through a caller-supplied
// all-gather of host bytes instead of NCCL (tests: several processes sharing one GPU, where NCCL refuses
// duplicate devices).  Every device-side exchange step then becomes stream sync + host all-gather; the
// peer-memory path (CUDA IPC mappings + the product kernels' peer stores) is unchanged, and no kernel ever
// waits on another process's kernel (the barrier is a host sync + the callback).
typedef int (*HostAllGather)(const void* send, void* recv, size_t bytes, void* user);

struct CommCtx {
  ncclComm_t comm = nullptr;
  HostAllGather host_fn = nullptr;
  void* host_user = nullptr;
  int rank = 0, nranks = 1;
  cudaStream_t cst = nullptr;          // communication stream (pack / all-gather / unpack)
  std::vector<cudaEvent_t> ev;         // chunk-ready events (compute -> comm), + 1 "exchange done" (comm -> compute)
  // peer-memory exchange: every rank's workspace mapped into this process (CUDA IPC over NVLink)
  std::vector<std::array<uint8_t, 96>> keys;   // [rank] -> (IPC handle, offset, size) the mappings belong to
  std::vector<uint8_t*> peer_ws;       // [rank] -> that rank's workspace (own entry: local pointer)
  std::vector<void*> opened;           // IPC mappings to close
  bool p2p = false;
  bool valid = false;                  // keys / peer_ws / p2p describe the current mappings
};

typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn get_addr_range() {
  static AddrRangeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<AddrRangeFn>(p);
  }
  return fn;
}

void close_peers(CommCtx& cc) {
  for (void* p : cc.opened) cudaIpcCloseMemHandle(p);
  cc.opened.clear();
  cc.peer_ws.clear();
  cc.keys.clear();
  cc.p2p = false;
  cc.valid = false;
}

// All-gather of `bytes` HOST bytes per rank (recv: nranks * bytes, rank order).  dscratch: device scratch of
// (nranks + 1) * bytes for the NCCL path.  Synchronises `st`.
ns_status_t comm_allgather_host(CommCtx& cc, const void* send, void* recv, size_t bytes, uint8_t* dscratch,
                                cudaStream_t st) {
  if (cc.nranks == 1) {
    memcpy(recv, send, bytes);
    return NS_OK;
  }
  if (cc.host_fn) {
    NS_CUDA(cudaStreamSynchronize(st));
    if (cc.host_fn(send, recv, bytes, cc.host_user) != 0) return fail(NS_ERR_NCCL, "host all-gather callback failed");
    return NS_OK;
  }
  NS_CUDA(cudaMemcpyAsync(dscratch, send, bytes, cudaMemcpyHostToDevice, st));
  NS_NCCL(ncclAllGather(dscratch, dscratch + bytes, bytes, ncclUint8, cc.comm, st));
  NS_CUDA(cudaMemcpyAsync(recv, dscratch + bytes, bytes * cc.nranks, cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  return NS_OK;
}

// All-gather of DEVICE buffers (ncclAllGather semantics: recv holds nranks * bytes in rank order; in place
// when send == recv + rank * bytes), enqueued on `st`.  Host control plane: staged through host memory.
ns_status_t comm_allgather_dev(CommCtx& cc, const void* dsend, void* drecv, size_t bytes, cudaStream_t st) {
  if (cc.host_fn) {
    std::vector<uint8_t> hs(bytes), hr(bytes * (size_t)cc.nranks);
    NS_CUDA(cudaMemcpyAsync(hs.data(), dsend, bytes, cudaMemcpyDeviceToHost, st));
    NS_CUDA(cudaStreamSynchronize(st));
    if (cc.host_fn(hs.data(), hr.data(), bytes, cc.host_user) != 0)
      return fail(NS_ERR_NCCL, "host all-gather callback failed");
    NS_CUDA(cudaMemcpyAsync(drecv, hr.data(), hr.size(), cudaMemcpyHostToDevice, st));
    NS_CUDA(cudaStreamSynchronize(st));
    return NS_OK;
  }
  NS_NCCL(ncclAllGather(dsend, drecv, bytes, ncclUint8, cc.comm, st));
  return NS_OK;
}

// Cross-rank barrier in stream order: every rank's work enqueued on its `st` before this point (including its
// kernels' peer stores, made visible by __threadfence_system) is complete before anything after it runs.
// NCCL: a one-double all-reduce on the stream; host control plane: stream sync + a one-byte all-gather.
ns_status_t comm_barrier(CommCtx& cc, double* dscratch, cudaStream_t st) {
  if (cc.nranks == 1) return NS_OK;
  if (cc.host_fn) {
    NS_CUDA(cudaStreamSynchronize(st));
    uint8_t b = 1;
    std::vector<uint8_t> all(cc.nranks);
    if (cc.host_fn(&b, all.data(), 1, cc.host_user) != 0) return fail(NS_ERR_NCCL, "host barrier callback failed");
    return NS_OK;
  }
  NS_NCCL(ncclAllReduce(dscratch, dscratch, 1, ncclDouble, ncclSum, cc.comm, st));
  return NS_OK;
}

// Map every rank's workspace into this process (collective, on EVERY call).  Each rank all-gathers its record
// (IPC handle of the allocation holding ws, ws's offset in it, the allocation size, "can export"); since all
// ranks see the same gathered records, the decision to reuse the cached mappings (every rank's record equals
// the one the mappings were opened for) or to re-open them is identical on every rank -- a workspace that
// moved on one rank only, or a peer that re-allocated, re-maps everywhere instead of desynchronising the
// collectives or storing through stale mappings.  All ranks take the peer-memory path only if every rank could
// export and open (torch's caching-allocator memory can be IPC-exported; VMM/expandable segments cannot), else
// the NCCL all-gather path everywhere.  NS_SHARD_P2P=0 forces the NCCL path.
// The gather also serves as the call's entry barrier: no rank stores into a peer before that peer has finished
// its previous call (its copy-out precedes its contribution in stream order).
ns_status_t setup_peers(CommCtx& cc, uint8_t* ws, uint8_t* scratch, cudaStream_t st) {
  static const bool allow = [] {
    const char* e = getenv("NS_SHARD_P2P");
    return !(e && e[0] == '0');
  }();
  const int nranks = cc.nranks, rank = cc.rank;
  if (nranks == 1) {
    if (!cc.valid || cc.peer_ws.size() != 1 || cc.peer_ws[0] != ws) {
      close_peers(cc);
      cc.peer_ws.assign(1, ws);
      cc.keys.assign(1, {});
      cc.p2p = allow;
      cc.valid = true;
    }
    return NS_OK;
  }
  struct Rec {
    cudaIpcMemHandle_t h;              // 64 bytes
    unsigned long long off, size;      // 16
    int ok;
    int pad0;
    unsigned long long ws_addr;        // the rank's workspace address: part of the key also without a handle
    int pad[8];
  };
  static_assert(sizeof(Rec) == 128, "IPC record size");
  Rec mine{};
  mine.ok = allow ? 1 : 0;
  CUdeviceptr base = 0;
  size_t size = 0;
  AddrRangeFn rng = get_addr_range();
  if (mine.ok && (!rng || rng(&base, &size, reinterpret_cast<CUdeviceptr>(ws)) != CUDA_SUCCESS)) mine.ok = 0;
  if (mine.ok && cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    mine.ok = 0;
  }
  mine.off = mine.ok ? (unsigned long long)(reinterpret_cast<uintptr_t>(ws) - (uintptr_t)base) : 0ull;
  mine.size = mine.ok ? (unsigned long long)size : 0ull;
  mine.ws_addr = (unsigned long long)reinterpret_cast<uintptr_t>(ws);
  std::vector<Rec> all(nranks);
  ns_status_t s = comm_allgather_host(cc, &mine, all.data(), sizeof(Rec), scratch, st);
  if (s != NS_OK) return s;
  auto key_of = [](const Rec& r) {
    std::array<uint8_t, 96> k{};
    memcpy(k.data(), &r, 96);          // handle, off, size, ok, ws address
    return k;
  };
  // decided on gathered data only (identical on every rank): the previous records of EVERY rank equal the
  // new ones, and so does this rank's own (which includes its ws address)
  bool same = cc.valid && (int)cc.keys.size() == nranks;
  for (int r = 0; r < nranks && same; ++r) same = (cc.keys[r] == key_of(all[r]));
  if (same) return NS_OK;              // identical decision on every rank (same gathered records)
  close_peers(cc);
  cc.peer_ws.assign(nranks, nullptr);
  cc.peer_ws[rank] = ws;
  int ok = 1;
  for (const Rec& r : all) ok &= r.ok;
  if (ok) {
    for (int r = 0; r < nranks && ok; ++r) {
      if (r == rank) continue;
      void* p = nullptr;
      if (cudaIpcOpenMemHandle(&p, all[r].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
        cudaGetLastError();
        ok = 0;
        break;
      }
      cc.opened.push_back(p);
      cc.peer_ws[r] = static_cast<uint8_t*>(p) + all[r].off;
    }
  }
  // agree on the outcome (an open can fail on one rank only)
  std::vector<int> oks(nranks);
  s = comm_allgather_host(cc, &ok, oks.data(), sizeof(int), scratch, st);
  if (s != NS_OK) return s;
  int all_ok = 1;
  for (int v : oks) all_ok &= v;
  cc.p2p = all_ok != 0;
  if (!cc.p2p) {
    for (void* p : cc.opened) cudaIpcCloseMemHandle(p);
    cc.opened.clear();
  }
  cc.keys.resize(nranks);
  for (int r = 0; r < nranks; ++r) cc.keys[r] = key_of(all[r]);
  cc.valid = true;
  return NS_OK;
}

// Mirror mode of the peer-store epilogue: 0 = receiver mirrors (default: each rank sends only the upper tile,
// half the NVLink bytes; a local transpose pass after the barrier), 1 = sender stores the mirror too.
int shard_sender_mirror() {
  static const int v = [] {
    const char* e = getenv("NS_SHARD_MIRROR");
    return (e && (e[0] == 's' || e[0] == '1')) ? 1 : 0;
  }();
  return v;
}

// One sharded run.  H_full != nullptr: every rank passes the full H (upper triangle read) and forms X_0 locally.
// Otherwise rows mode: H_rows holds rows [r0, r1) of H; X_0 is assembled on every rank from all ranks' rows
// (peer stores from ns_init_rows_kernel, or an all-gather of the row panels on the NCCL path) and the rank
// receives rows [r0, r1) of R in R (ldr).
ns_status_t run_sharded(CommCtx& cc, const ShardLayout& SL, uint8_t* ws, const double* H_full, const double* H_rows,
                        long long ldh, long long r0, long long r1, const JobParams& jp, int32_t max_steps, double tol,
                        ns_tolmode_t tm, double* R, long long ldr, cudaStream_t st, DevState& out_state,
                        int* launches, int sender_mirror) {
  const Layout& L = SL.base;
  double* Xa = reinterpret_cast<double*>(ws + L.off_xa);
  double* Xb = reinterpret_cast<double*>(ws + L.off_xb);
  double* Y = reinterpret_cast<double*>(ws + L.off_y);
  double* res = reinterpret_cast<double*>(ws + L.off_res);
  double* trp = reinterpret_cast<double*>(ws + L.off_tr);
  int2* tiles = reinterpret_cast<int2*>(ws + L.off_tiles);
  int2* my = reinterpret_cast<int2*>(ws + SL.off_my);
  double* send = reinterpret_cast<double*>(ws + SL.off_send);
  double* recv = reinterpret_cast<double*>(ws + SL.off_recv);
  double* rsend = reinterpret_cast<double*>(ws + SL.off_rsend);
  double* rrecv = reinterpret_cast<double*>(ws + SL.off_rrecv);
  JobParams* djobs = reinterpret_cast<JobParams*>(ws + L.off_jobs);
  DevState* state = reinterpret_cast<DevState*>(ws + L.off_state);
  int* n_active = reinterpret_cast<int*>(ws + L.off_active);
  HostRing& rg = ring();
  if (!rg.ok) return fail(NS_ERR_CUDA, "pinned status ring allocation failed");

  // entry: the collective peer-mapping check (also the entry barrier, see setup_peers)
  ns_status_t ps = setup_peers(cc, ws, ws + SL.off_ipc, st);
  if (ps != NS_OK) return ps;
  const bool p2p = cc.p2p;

  std::vector<int2> tl = make_tiles(L.n);
  std::vector<int2> mt = shard_tiles(tl, SL.nranks, SL.rank);
  NS_CUDA(cudaMemcpyAsync(tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  if (!mt.empty()) NS_CUDA(cudaMemcpyAsync(my, mt.data(), mt.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
  NS_CUDA(cudaMemcpyAsync(djobs, &jp, sizeof(JobParams), cudaMemcpyHostToDevice, st));
  CUtensorMap tmA, tmB, tmY;
  ns_status_t s;
  if ((s = encode_map(&tmA, Xa, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map(&tmB, Xb, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map(&tmY, Y, L.d_pad, 1)) != NS_OK) return s;

  const size_t tile_elems = (size_t)kTile * kTile;
  const size_t chunk_elems = (size_t)SL.cs * tile_elems;          // doubles per rank per chunk
  const int n_my = (int)mt.size();
  while (cc.ev.size() < (size_t)SL.n_chunks + 1) {
    cudaEvent_t e;
    NS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cc.ev.push_back(e);
  }
  int nl = 0;
  // NCCL fallback: one symmetric product on the rank's tiles, chunk by chunk, with the exchange of chunk c on
  // the communication stream overlapping the computation of chunk c+1.
  auto product_and_exchange = [&](const CUtensorMap& tP, const CUtensorMap& tQ, double* C, const double* Xold,
                                  double* partial, int mode) -> ns_status_t {
    for (int c = 0; c < SL.n_chunks; ++c) {
      const int s0 = c * SL.cs;
      const int cnt = std::max(0, std::min(SL.cs, n_my - s0));
      if (cnt > 0) {
        // mode 0: residual partial per local tile slot; mode 1: trace partial per diagonal block I (global
        // index: an offset by s0 would write past the n-entry trace buffer)
        ProdParams pp{my + s0, cnt, L.d_pad / kBK, L.d, L.d_pad, (long long)L.d_pad * L.d_pad, C, Xold,
                      mode == 0 ? partial + s0 : partial, state, mode};
        NS_CUDA(launch_product(tP, tQ, pp, 1, st));
        nl += 1;
      }
      NS_CUDA(cudaEventRecord(cc.ev[c], st));
      NS_CUDA(cudaStreamWaitEvent(cc.cst, cc.ev[c], 0));
      if (cnt > 0) NS_CUDA(launch_pack_tiles(C, my + s0, cnt, send + (size_t)s0 * tile_elems, L.d_pad, cc.cst));
      ns_status_t e = comm_allgather_dev(cc, send + (size_t)s0 * tile_elems, recv + (size_t)c * SL.nranks * chunk_elems,
                                         chunk_elems * sizeof(double), cc.cst);
      if (e != NS_OK) return e;
      NS_CUDA(launch_unpack_tiles(C, tiles, L.n_tiles, recv + (size_t)c * SL.nranks * chunk_elems, SL.cs, s0,
                                  SL.nranks, SL.rank, L.d_pad, cc.cst));
      nl += 2;
    }
    NS_CUDA(cudaEventRecord(cc.ev[SL.n_chunks], cc.cst));
    NS_CUDA(cudaStreamWaitEvent(st, cc.ev[SL.n_chunks], 0));
    return NS_OK;
  };

  // Peer-memory exchange (default): the product kernel's epilogue stores each tile (and, in sender-mirror mode,
  // its mirror) plus its residual / trace partial straight into every rank's buffers through the IPC mappings,
  // so the exchange rides on the contraction tile by tile; one tiny all-reduce per product is the cross-rank
  // barrier (all peers' stores done) before anything reads the full matrix; in receiver-mirror mode each rank
  // then fills the lower halves of its peers' tiles locally.
  // [7][P]: Y, Xa, Xb, res, tr (even steps), tr (odd steps), Xa again (init targets).  The trace partials
  // alternate by step parity: a fast rank's update j (writing tr X_{j+1}) may overlap a slow rank's decide j.
  double** dptr = reinterpret_cast<double**>(ws + SL.off_ptrs);
  if (p2p) {
    std::vector<double*> h(6 * (size_t)SL.nranks);
    for (int r = 0; r < SL.nranks; ++r) {
      uint8_t* w = cc.peer_ws[r];
      h[0 * SL.nranks + r] = reinterpret_cast<double*>(w + L.off_y);
      h[1 * SL.nranks + r] = reinterpret_cast<double*>(w + L.off_xa);
      h[2 * SL.nranks + r] = reinterpret_cast<double*>(w + L.off_xb);
      h[3 * SL.nranks + r] = reinterpret_cast<double*>(w + L.off_res);
      h[4 * SL.nranks + r] = reinterpret_cast<double*>(w + L.off_tr);
      h[5 * SL.nranks + r] = reinterpret_cast<double*>(w + L.off_tr) + L.n;
    }
    NS_CUDA(cudaMemcpyAsync(dptr, h.data(), h.size() * sizeof(double*), cudaMemcpyHostToDevice, st));
  }
  Profiler& pf = prof();
  int n_prof = 0;                      // event pairs recorded (kernel only, not the barrier)
  std::vector<int> prof_mode;
  auto product_p2p = [&](const CUtensorMap& tP, const CUtensorMap& tQ, double* C, int which_c, const double* Xold,
                         double* partial, int which_part, int mode) -> ns_status_t {
    if (pf.on) NS_CUDA(cudaEventRecord(pf.get(2 * n_prof), st));
    if (n_my > 0) {
      ProdParams pp{my, n_my, L.d_pad / kBK, L.d, L.d_pad, (long long)L.d_pad * L.d_pad, C, Xold, partial, state, mode};
      pp.dst = dptr + (size_t)which_c * SL.nranks;
      pp.dst_part = dptr + (size_t)which_part * SL.nranks;
      pp.n_dst = SL.nranks;
      pp.gt_off = SL.rank;
      pp.gt_stride = SL.nranks;
      pp.n_tiles_total = L.n_tiles;
      pp.remote_mirror = sender_mirror;
      NS_CUDA(launch_product(tP, tQ, pp, 1, st));
      nl += 1;
    }
    if (pf.on) {
      NS_CUDA(cudaEventRecord(pf.get(2 * n_prof + 1), st));
      prof_mode.push_back(mode);
      ++n_prof;
    }
    ns_status_t e = comm_barrier(cc, rsend, st);
    if (e != NS_OK) return e;
    if (!sender_mirror && SL.nranks > 1) {
      NS_CUDA(launch_mirror_remote(C, tiles, L.n_tiles, SL.nranks, SL.rank, L.d_pad, st));
      nl += 1;
    }
    return NS_OK;
  };

  NS_CUDA(launch_zero_state(state, 1, n_active, st));
  nl += 1;
  if (H_full) {
    NS_CUDA(launch_init(H_full, ldh, 0, Xa, djobs, L.d, L.d_pad, 1, st));
    nl += 1;
  } else if (p2p) {
    // every rank stores its rows' upper parts and their mirrors into every rank's X_0; the padding (never
    // written remotely) is zeroed locally
    if (L.d_pad > L.d) {
      NS_CUDA(cudaMemset2DAsync(Xa + L.d, (size_t)L.d_pad * 8, 0, (size_t)(L.d_pad - L.d) * 8, (size_t)L.d, st));
      NS_CUDA(cudaMemsetAsync(Xa + (size_t)L.d * L.d_pad, 0, (size_t)(L.d_pad - L.d) * L.d_pad * 8, st));
    }
    NS_CUDA(launch_init_rows(H_rows, ldh, r0, r1, dptr + 1 * (size_t)SL.nranks, SL.nranks, jp.s, jp.alpha, L.d,
                             L.d_pad, st));
    nl += 1;
    ns_status_t e = comm_barrier(cc, rsend, st);
    if (e != NS_OK) return e;
  } else {
    // NCCL path: all-gather the row panels of H into Y (free until the first square), then form X_0 locally
    const long long rows = r1 - r0;
    if (rows > 0)
      NS_CUDA(cudaMemcpy2DAsync(Y + (size_t)r0 * L.d_pad, (size_t)L.d_pad * 8, H_rows, (size_t)ldh * 8, (size_t)L.d * 8,
                                (size_t)rows, cudaMemcpyDeviceToDevice, st));
    ns_status_t e = comm_allgather_dev(cc, Y + (size_t)r0 * L.d_pad, Y, (size_t)rows * L.d_pad * sizeof(double), st);
    if (e != NS_OK) return e;
    NS_CUDA(launch_init(Y, L.d_pad, 0, Xa, djobs, L.d, L.d_pad, 1, st));
    nl += 1;
  }
  NS_CUDA(launch_trace_partials(Xa, L.d, L.d_pad, 1, trp, st));
  nl += 1;
  LoopParams lp{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0};
  const int LA = 2;
  for (int j = 0; j <= max_steps; ++j) {
    if (j >= LA) {
      const int slot = (j - LA) % 16;
      NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
      if (rg.slots[slot] == 0) break;   // identical on every rank: decisions use identical bits
    }
    const bool odd = (j & 1) != 0;
    double* Xc = odd ? Xb : Xa;
    double* Xn = odd ? Xa : Xb;
    const CUtensorMap& tmC = odd ? tmB : tmA;
    if (p2p) {
      // Y tiles of this rank into every rank's Y (+ residual partials into every rank's res, global slots)
      ns_status_t e1 = product_p2p(tmC, tmC, Y, 0, nullptr, res, 3, 0);
      if (e1 != NS_OK) return e1;
      NS_CUDA(launch_decide(state, djobs, res, L.n_tiles, trp + (odd ? L.n : 0), L.n, lp, 1, n_active, st));
      nl += 1;
      if (j < max_steps) {
        // X_{j+1} tiles into every rank's X_{j+1}; the diagonal tiles' trace partials likewise (other parity)
        ns_status_t e2 = product_p2p(tmC, tmY, Xn, odd ? 1 : 2, Xc, trp + (odd ? 0 : L.n), odd ? 4 : 5, 1);
        if (e2 != NS_OK) return e2;
      }
    } else {
      // own Y tiles (chunked, exchange overlapped) + residual sum of the rank's tiles
      ns_status_t e1 = product_and_exchange(tmC, tmC, Y, nullptr, res, 0);
      if (e1 != NS_OK) return e1;
      NS_CUDA(launch_shard_sum(res, n_my, rsend, st));
      e1 = comm_allgather_dev(cc, rsend, rrecv, sizeof(double), st);
      if (e1 != NS_OK) return e1;
      // decide (identical on all ranks)
      NS_CUDA(launch_decide(state, djobs, res, 0, trp, L.n, lp, 1, n_active, st, rrecv, SL.nranks));
      nl += 2;
      if (j < max_steps) {
        ns_status_t e2 = product_and_exchange(tmC, tmY, Xn, Xc, trp, 1);
        if (e2 != NS_OK) return e2;
        NS_CUDA(launch_trace_partials(Xn, L.d, L.d_pad, 1, trp, st));
        nl += 1;
      }
    }
    NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], n_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
  }
  if (H_full) NS_CUDA(launch_copy_out(Xa, Xb, L.d, L.d_pad, state, R, ldr, 0, 1, st));
  else NS_CUDA(launch_copy_out(Xa, Xb, L.d, L.d_pad, state, R, ldr, 0, 1, st, (int)r0, (int)(r1 - r0)));
  nl += 1;
  NS_CUDA(cudaMemcpyAsync(&out_state, state, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  if (launches) *launches = nl;
  if (pf.on) {   // products that did work: squares 0..j, updates 0..j-1 (launches past the stop exit at once)
    int sq = 0, up = 0;
    for (int q = 0; q < n_prof; ++q) {
      const bool is_sq = prof_mode[q] == 0;
      if (is_sq ? sq > out_state.j : up >= out_state.j) continue;
      float ms = 0.f;
      NS_CUDA(cudaEventElapsedTime(&ms, pf.get(2 * q), pf.get(2 * q + 1)));
      if (is_sq) {
        pf.acc.ms_square += ms;
        pf.acc.n_square += 1;
        ++sq;
      } else {
        pf.acc.ms_update += ms;
        pf.acc.n_update += 1;
        ++up;
      }
    }
    pf.acc.n_calls += 1;
  }
  return NS_OK;
}

// The sharded algorithm with P ranks emulated on ONE GPU (tests): P workspace replicas side by side,
// each rank's product kernel launched in turn on one stream with the same peer-store epilogue as the
// multi-GPU path (destinations: all replicas), every replica running its own decide.  No kernel waits
// on another (stream order replaces the cross-rank barrier), so this is safe on one device; it checks
// the partitioning, the global partial slots, the trace-parity buffers and that all ranks take
// identical decisions (their final states must agree bit for bit).
// flags: bit 0 = block-row input (replica r forms its share of X_0 from rows [r d/P, (r+1) d/P) of H with the
// rows entry's init kernel, storing into every replica); bit 1 = sender-mirror epilogue (default: receivers mirror).
ns_status_t run_sharded_emulated(int64_t d, int P, uint8_t* ws, size_t stride, const double* H, long long ldh,
                                 const JobParams& jp, int32_t max_steps, double tol, ns_tolmode_t tm, double* R,
                                 long long ldr, cudaStream_t st, DevState& out_state, int* launches, int flags) {
  const bool rows_mode = (flags & 1) != 0;
  const int sender_mirror = (flags & 2) ? 1 : 0;
  std::vector<ShardLayout> sl;
  std::vector<uint8_t*> w(P);
  for (int r = 0; r < P; ++r) {
    sl.push_back(make_shard_layout(d, P, r));
    w[r] = ws + (size_t)r * stride;
  }
  const Layout& L = sl[0].base;
  auto ptr = [&](int r, size_t off) { return reinterpret_cast<double*>(w[r] + off); };
  HostRing& rg = ring();
  if (!rg.ok) return fail(NS_ERR_CUDA, "pinned status ring allocation failed");
  const std::vector<int2> tl = make_tiles(L.n);
  std::vector<std::vector<int2>> mt(P);
  std::vector<CUtensorMap> tA(P), tB(P), tY(P);
  ns_status_t s;
  // peer pointer table [6][P] (Y, Xa, Xb, res, tr even, tr odd), identical for every replica; replica 0 holds it
  double** dptr = reinterpret_cast<double**>(w[0] + sl[0].off_ptrs);
  std::vector<double*> h(6 * (size_t)P);
  for (int r = 0; r < P; ++r) {
    h[0 * P + r] = ptr(r, L.off_y);
    h[1 * P + r] = ptr(r, L.off_xa);
    h[2 * P + r] = ptr(r, L.off_xb);
    h[3 * P + r] = ptr(r, L.off_res);
    h[4 * P + r] = ptr(r, L.off_tr);
    h[5 * P + r] = ptr(r, L.off_tr) + L.n;
  }
  NS_CUDA(cudaMemcpyAsync(dptr, h.data(), h.size() * sizeof(double*), cudaMemcpyHostToDevice, st));
  int nl = 0;
  for (int r = 0; r < P; ++r) {
    NS_CUDA(cudaMemcpyAsync(w[r] + L.off_tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    mt[r] = shard_tiles(tl, P, r);
    int2* my = reinterpret_cast<int2*>(w[r] + sl[r].off_my);
    if (!mt[r].empty()) NS_CUDA(cudaMemcpyAsync(my, mt[r].data(), mt[r].size() * sizeof(int2), cudaMemcpyHostToDevice, st));
    NS_CUDA(cudaMemcpyAsync(w[r] + L.off_jobs, &jp, sizeof(JobParams), cudaMemcpyHostToDevice, st));
    if ((s = encode_map(&tA[r], ptr(r, L.off_xa), L.d_pad, 1)) != NS_OK) return s;
    if ((s = encode_map(&tB[r], ptr(r, L.off_xb), L.d_pad, 1)) != NS_OK) return s;
    if ((s = encode_map(&tY[r], ptr(r, L.off_y), L.d_pad, 1)) != NS_OK) return s;
    DevState* state = reinterpret_cast<DevState*>(w[r] + L.off_state);
    int* n_active = reinterpret_cast<int*>(w[r] + L.off_active);
    NS_CUDA(launch_zero_state(state, 1, n_active, st));
    nl += 1;
    if (!rows_mode) {
      NS_CUDA(launch_init(H, ldh, 0, ptr(r, L.off_xa), reinterpret_cast<JobParams*>(w[r] + L.off_jobs), L.d, L.d_pad, 1, st));
      nl += 1;
    } else if (L.d_pad > L.d) {
      double* Xa = ptr(r, L.off_xa);
      NS_CUDA(cudaMemset2DAsync(Xa + L.d, (size_t)L.d_pad * 8, 0, (size_t)(L.d_pad - L.d) * 8, (size_t)L.d, st));
      NS_CUDA(cudaMemsetAsync(Xa + (size_t)L.d * L.d_pad, 0, (size_t)(L.d_pad - L.d) * L.d_pad * 8, st));
    }
  }
  if (rows_mode) {   // each replica's row panel into every replica's X_0 (the rows entry's peer-store init)
    for (int r = 0; r < P; ++r) {
      const long long r0 = d * r / P, r1 = d * (r + 1) / P;
      NS_CUDA(launch_init_rows(H + r0 * ldh, ldh, r0, r1, dptr + 1 * (size_t)P, P, jp.s, jp.alpha, L.d, L.d_pad, st));
      nl += 1;
    }
  }
  for (int r = 0; r < P; ++r) {
    NS_CUDA(launch_trace_partials(ptr(r, L.off_xa), L.d, L.d_pad, 1, ptr(r, L.off_tr), st));
    nl += 1;
  }
  auto products = [&](bool odd, int mode) -> ns_status_t {
    for (int r = 0; r < P; ++r) {
      if (mt[r].empty()) continue;
      const CUtensorMap& tC = odd ? tB[r] : tA[r];
      double* Xc = ptr(r, odd ? L.off_xb : L.off_xa);
      double* C = (mode == 0) ? ptr(r, L.off_y) : ptr(r, odd ? L.off_xa : L.off_xb);
      ProdParams pp{reinterpret_cast<int2*>(w[r] + sl[r].off_my), (int)mt[r].size(), L.d_pad / kBK, L.d, L.d_pad,
                    (long long)L.d_pad * L.d_pad, C, mode == 1 ? Xc : nullptr,
                    mode == 0 ? ptr(r, L.off_res) : ptr(r, L.off_tr) + (odd ? 0 : L.n),
                    reinterpret_cast<DevState*>(w[r] + L.off_state), mode};
      const int which_c = (mode == 0) ? 0 : (odd ? 1 : 2);
      const int which_p = (mode == 0) ? 3 : (odd ? 4 : 5);
      pp.dst = dptr + (size_t)which_c * P;
      pp.dst_part = dptr + (size_t)which_p * P;
      pp.n_dst = P;
      pp.gt_off = r;
      pp.gt_stride = P;
      pp.n_tiles_total = L.n_tiles;
      pp.remote_mirror = sender_mirror;
      NS_CUDA(launch_product(tC, mode == 0 ? tC : tY[r], pp, 1, st));
      nl += 1;
    }
    // (stream order is the barrier) receivers mirror their peers' tiles
    if (!sender_mirror && P > 1)
      for (int r = 0; r < P; ++r) {
        double* C = (mode == 0) ? ptr(r, L.off_y) : ptr(r, odd ? L.off_xa : L.off_xb);
        NS_CUDA(launch_mirror_remote(C, reinterpret_cast<int2*>(w[r] + L.off_tiles), L.n_tiles, P, r, L.d_pad, st));
        nl += 1;
      }
    return NS_OK;
  };
  LoopParams lp{L.d, L.d_pad, max_steps, (int)tm, tol, 0.0, -1, 0};
  const int LA = 2;
  for (int j = 0; j <= max_steps; ++j) {
    if (j >= LA) {
      const int slot = (j - LA) % 16;
      NS_CUDA(cudaEventSynchronize(rg.ev[slot]));
      if (rg.slots[slot] == 0) break;
    }
    const bool odd = (j & 1) != 0;
    if ((s = products(odd, 0)) != NS_OK) return s;
    for (int r = 0; r < P; ++r) {
      NS_CUDA(launch_decide(reinterpret_cast<DevState*>(w[r] + L.off_state), reinterpret_cast<JobParams*>(w[r] + L.off_jobs),
                            ptr(r, L.off_res), L.n_tiles, ptr(r, L.off_tr) + (odd ? L.n : 0), L.n, lp, 1,
                            reinterpret_cast<int*>(w[r] + L.off_active), st));
      nl += 1;
    }
    if (j < max_steps && (s = products(odd, 1)) != NS_OK) return s;
    NS_CUDA(cudaMemcpyAsync(&rg.slots[j % 16], w[0] + L.off_active, sizeof(int), cudaMemcpyDeviceToHost, st));
    NS_CUDA(cudaEventRecord(rg.ev[j % 16], st));
  }
  if (!rows_mode) {
    NS_CUDA(launch_copy_out(ptr(0, L.off_xa), ptr(0, L.off_xb), L.d, L.d_pad,
                            reinterpret_cast<DevState*>(w[0] + L.off_state), R, ldr, 0, 1, st));
    nl += 1;
  } else {   // every replica writes its own row block of R (the rows entry's output)
    for (int r = 0; r < P; ++r) {
      const long long r0 = d * r / P, r1 = d * (r + 1) / P;
      NS_CUDA(launch_copy_out(ptr(r, L.off_xa), ptr(r, L.off_xb), L.d, L.d_pad,
                              reinterpret_cast<DevState*>(w[r] + L.off_state), R + r0 * ldr, ldr, 0, 1, st, (int)r0,
                              (int)(r1 - r0)));
      nl += 1;
    }
  }
  std::vector<DevState> states(P);
  for (int r = 0; r < P; ++r)
    NS_CUDA(cudaMemcpyAsync(&states[r], w[r] + L.off_state, sizeof(DevState), cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  for (int r = 1; r < P; ++r)
    if (memcmp(&states[r], &states[0], sizeof(DevState)) != 0)
      return fail(NS_ERR_CUDA, "emulated ranks diverged (rank %d state differs from rank 0)", r);
  out_state = states[0];
  if (launches) *launches = nl;
  return NS_OK;
}

// alpha = ||H - sI||_inf on the device (the Gershgorin bound of ns_scale_bound, N1), read back with one
// 8-byte copy; scratch: d + 1 doubles of device memory that the caller's next launches overwrite anyway.
ns_status_t device_scale_bound(const double* H, long long ldh, int d, double s, double* scratch, cudaStream_t st,
                               double* alpha) {
  NS_CUDA(launch_scale_bound(H, ldh, d, s, scratch, scratch + d, st));
  NS_CUDA(cudaMemcpyAsync(alpha, scratch + d, sizeof(double), cudaMemcpyDeviceToHost, st));
  NS_CUDA(cudaStreamSynchronize(st));
  if (!std::isfinite(*alpha)) return fail(NS_ERR_INVALID_ARG, "H - sI has a non-finite entry: no scale bound");
  if (!(*alpha > 0.0)) *alpha = 1.0;       // H = sI: X_0 = 0 for any alpha
  return NS_OK;
}

void fill_result(const DevState& s, int launches, ns_result_t* out) {
  out->kernel_launches = launches;
  out->switch_step = s.sw_step;
  out->pre_polish_residual = s.sw ? s.sw_residual : 0.0;
  out->steps = s.j;
  out->flags = s.flags;
  out->residual = s.residual;
  out->trace = s.trace;
  out->index_cert = s.cert;
}

}  // namespace

extern "C" {

size_t ns_workspace_bytes(int64_t d, ns_precision_t prec) {
  if (d < 1) return 0;
  const bool mixed = prec == NS_PREC_MIXED_BF16X3 || prec == NS_PREC_MIXED_TF32X3;
  // the mixed layout carries the Ozaki buffers too (options.polish = 1)
  return make_layout(d, 1, mixed, prec == NS_PREC_FP64_OZAKI || mixed, prec == NS_PREC_MIXED_TF32X3).total;
}

size_t ns_workspace_bytes_batched(int64_t d, int64_t batch, ns_precision_t prec) {
  if (d < 1 || batch < 1) return 0;
  return make_layout(d, batch, false, prec == NS_PREC_FP64_OZAKI).total;
}

size_t ns_workspace_bytes_host(int64_t d, ns_precision_t prec) { return ns_workspace_bytes(d, prec); }

size_t ns_workspace_bytes_ex(int64_t d, ns_precision_t prec, const ns_options_t* opts) {
  if (d < 1) return 0;
  const size_t base = ns_workspace_bytes(d, prec);
  if (!opts || !to_opts(opts).general_filter()) return base;
  const size_t dp = (size_t)((d + kTile - 1) / kTile * kTile);
  return align256(base) + align256(dp * dp * sizeof(double));   // + E, the Horner buffer of run_filter
}

void ns_options_default(ns_options_t* o) {
  if (!o) return;
  *o = ns_options_t{};
  o->switch_tol = 1e-3;
  o->cg_iters = 512;
  o->stop_at_switch = 0;
  o->lookahead = 0;
  o->polish = 2;
  o->filter_a = 1.5;
  o->filter_b = -0.5;
}

ns_status_t ns_reflector_ex(const double* H, int64_t d, int64_t ldh, double s, double alpha, int32_t k,
                            int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec, double* R,
                            int64_t ldr, void* ws, size_t ws_bytes, void* stream, const ns_options_t* opts,
                            ns_result_t* out) {
  g_last_error.clear();
  ns_status_t st = check_common(d, max_steps, tol, tm, prec);
  if (st != NS_OK) return st;
  if (!H || !R || !ws || !out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (ldh < d || ldr < d) return fail(NS_ERR_INVALID_ARG, "leading dimensions must be >= d");
  if (!std::isfinite(s)) return fail(NS_ERR_INVALID_ARG, "shift s must be finite");
  if (!(alpha >= 0.0) || !std::isfinite(alpha))
    return fail(NS_ERR_INVALID_ARG, "alpha must be finite and > 0 (or 0: Gershgorin bound on the device)");
  if (k < 0 || k > d) return fail(NS_ERR_INVALID_ARG, "k must lie in [0, d]");
  if (R == H) return fail(NS_ERR_INVALID_ARG, "R must not alias H");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const bool tf32 = (prec == NS_PREC_MIXED_TF32X3);
  const bool mixed = (prec == NS_PREC_MIXED_BF16X3) || tf32;
  const bool ozaki = (prec == NS_PREC_FP64_OZAKI);
  if (ozaki && d > kOzMaxD) return fail(NS_ERR_UNSUPPORTED, "the Ozaki path needs d <= %d", kOzMaxD);
  const Layout L = make_layout(d, 1, mixed, ozaki || mixed, tf32);
  if (ws_bytes < L.total)
    return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  if (alpha == 0.0) {   // N1: alpha = ||H - sI||_inf >= ||H - sI||_2 from the device (Y is scratch until the first square)
    st = device_scale_bound(H, ldh, (int)d, s, reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + L.off_y),
                            static_cast<cudaStream_t>(stream), &alpha);
    if (st != NS_OK) return st;
  }
  out->alpha = alpha;
  const Opts o = to_opts(opts);
  if (mixed && (!(o.switch_tol >= 0.0) || o.cg_iters < 0 || o.polish < 0 || o.polish > 2))
    return fail(NS_ERR_INVALID_ARG, "bad mixed options");
  if (!std::isfinite(o.ca) || !std::isfinite(o.cb)) return fail(NS_ERR_INVALID_ARG, "filter coefficients must be finite");
  if (mixed && (o.ca != 1.5 || o.cb != -0.5))
    return fail(NS_ERR_UNSUPPORTED, "the mixed path runs the Newton-Schulz step (1.5, -0.5) only");
  for (double v : o.cz)
    if (!std::isfinite(v)) return fail(NS_ERR_INVALID_ARG, "filter coefficients must be finite");
  if (o.general_filter()) {   // N3: general odd polynomial filter (degree >= 5)
    if (mixed) return fail(NS_ERR_UNSUPPORTED, "general polynomial filters run on the FP64 and Ozaki paths");
    if (ws_bytes < ns_workspace_bytes_ex(d, prec, opts))
      return fail(NS_ERR_WORKSPACE, "workspace too small for a general filter: %zu < %zu bytes", ws_bytes,
                  ns_workspace_bytes_ex(d, prec, opts));
    DevState ds;
    int nl = 0;
    st = run_filter(L, static_cast<uint8_t*>(ws), H, ldh, JobParams{s, alpha, k, 0}, max_steps, tol, tm, R, ldr,
                    static_cast<cudaStream_t>(stream), o, ozaki, ds, &nl);
    xprof_flush();
    if (st != NS_OK) return st;
    fill_result(ds, nl, out);
    return NS_OK;
  }
  std::vector<JobParams> jobs{JobParams{s, alpha, k, 0}};
  int nl = 0;
  if (mixed || ozaki) {
    DevState ds;
    st = mixed ? run_mixed(L, static_cast<uint8_t*>(ws), H, ldh, jobs[0], max_steps, tol, tm, R, ldr,
                           static_cast<cudaStream_t>(stream), o, ds, &nl, tf32)
               : run_ozaki(L, static_cast<uint8_t*>(ws), H, ldh, jobs[0], max_steps, tol, tm, R, ldr,
                           static_cast<cudaStream_t>(stream), o, ds, &nl);
    xprof_flush();
    if (st != NS_OK) return st;
    fill_result(ds, nl, out);
    return NS_OK;
  }
  std::vector<DevState> states;
  st = run_loop(L, static_cast<uint8_t*>(ws), H, ldh, 0, jobs, max_steps, tol, tm, R, ldr, 0,
                static_cast<cudaStream_t>(stream), states, &nl, o);
  if (st != NS_OK) return st;
  fill_result(states[0], nl, out);
  return NS_OK;
}

ns_status_t ns_reflector(const double* H, int64_t d, int64_t ldh, double s, double alpha, int32_t k,
                         int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec, double* R, int64_t ldr,
                         void* ws, size_t ws_bytes, void* stream, ns_result_t* out) {
  return ns_reflector_ex(H, d, ldh, s, alpha, k, max_steps, tol, tm, prec, R, ldr, ws, ws_bytes, stream, nullptr,
                         out);
}

ns_status_t ns_reflector_host(const double* H_host, int64_t d, int64_t ldh, double s, double alpha, int32_t k,
                              int32_t max_steps, double tol, ns_tolmode_t tm, ns_precision_t prec, double* R_host,
                              int64_t ldr, void* ws, size_t ws_bytes, void* stream, ns_result_t* out) {
  g_last_error.clear();
  ns_status_t st = check_common(d, max_steps, tol, tm, prec);
  if (st != NS_OK) return st;
  if (!H_host || !R_host || !ws || !out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (ldh < d || ldr < d) return fail(NS_ERR_INVALID_ARG, "leading dimensions must be >= d");
  if (!std::isfinite(s)) return fail(NS_ERR_INVALID_ARG, "shift s must be finite");
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return fail(NS_ERR_INVALID_ARG, "alpha must be finite and > 0");
  if (k < 0 || k > d) return fail(NS_ERR_INVALID_ARG, "k must lie in [0, d]");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const bool tf32 = (prec == NS_PREC_MIXED_TF32X3);
  const bool mixed = (prec == NS_PREC_MIXED_BF16X3) || tf32;
  const bool ozaki = (prec == NS_PREC_FP64_OZAKI);
  if (ozaki && d > kOzMaxD) return fail(NS_ERR_UNSUPPORTED, "the Ozaki path needs d <= %d", kOzMaxD);
  const Layout L = make_layout(d, 1, mixed, ozaki || mixed, tf32);
  if (ws_bytes < L.total)
    return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  // H staged in the Y buffer (dead until the first square), R staged there after the loop.  FP64 path
  // with d >= 1024: run_loop stages H itself, in row chunks overlapped with the first square product.
  double* stage = reinterpret_cast<double*>(w + L.off_y);
  static const bool chunks_on = [] {
    const char* e = getenv("NS_H2D_CHUNKS");   // 0: stage H in one copy before the loop (A/B knob)
    return !(e && e[0] == '0');
  }();
  const bool fp64_chunked = chunks_on && !mixed && !ozaki && small_dpad(d) == 0 && d >= 1024 && spec_ctx().ok;
  if (!fp64_chunked)
    NS_CUDA(cudaMemcpy2DAsync(stage, (size_t)d * 8, H_host, (size_t)ldh * 8, (size_t)d * 8, (size_t)d,
                              cudaMemcpyHostToDevice, cs));
  std::vector<JobParams> jobs{JobParams{s, alpha, k, 0}};
  std::vector<DevState> states(1);
  int nl = 0;
  if (mixed) {
    st = run_mixed(L, w, stage, d, jobs[0], max_steps, tol, tm, stage, d, cs, Opts{}, states[0], &nl, tf32);
    xprof_flush();
  } else if (ozaki) {
    st = run_ozaki(L, w, stage, d, jobs[0], max_steps, tol, tm, stage, d, cs, Opts{}, states[0], &nl);
    xprof_flush();
  } else {
    // FP64 path: if R_host is pinned (device-accessible), the result may be copied speculatively
    // behind the last square product (run_loop); otherwise one D2H copy after the loop
    Opts o;
    bool hit = false;
    if (fp64_chunked) {
      o.h_host = H_host;
      o.h_ldh = ldh;
    }
    cudaPointerAttributes pa{};
    static const bool spec_on = [] {
      const char* e = getenv("NS_SPEC_COPY");   // 0: always copy R after the loop (A/B knob)
      return !(e && e[0] == '0');
    }();
    if (spec_on && cudaPointerGetAttributes(&pa, R_host) == cudaSuccess && pa.type == cudaMemoryTypeHost &&
        pa.devicePointer != nullptr) {
      o.spec_R = static_cast<double*>(pa.devicePointer);
      o.spec_ldr = ldr;
      o.spec_hit = &hit;
    } else {
      (void)cudaGetLastError();   // pageable memory: clear the query's error state
    }
    st = run_loop(L, w, stage, d, 0, jobs, max_steps, tol, tm, stage, d, 0, cs, states, &nl, o);
    if (st != NS_OK) return st;
    if (hit) {
      fill_result(states[0], nl, out);
      out->alpha = alpha;
      return NS_OK;
    }
  }
  if (st != NS_OK) return st;
  NS_CUDA(cudaMemcpy2DAsync(R_host, (size_t)ldr * 8, stage, (size_t)d * 8, (size_t)d * 8, (size_t)d,
                            cudaMemcpyDeviceToHost, cs));
  NS_CUDA(cudaStreamSynchronize(cs));
  fill_result(states[0], nl, out);
  out->alpha = alpha;
  return NS_OK;
}

ns_status_t ns_reflector_batched(const double* H, int64_t d, int64_t batch, int64_t stride_h, const double* s,
                                 const double* alpha, const int32_t* k, int32_t max_steps, double tol,
                                 ns_tolmode_t tm, ns_precision_t prec, double* R, int64_t stride_r, void* ws,
                                 size_t ws_bytes, void* stream, ns_result_t* outs) {
  g_last_error.clear();
  ns_status_t st = check_common(d, max_steps, tol, tm, prec);
  if (st != NS_OK) return st;
  if (prec != NS_PREC_FP64 && prec != NS_PREC_FP64_OZAKI)
    return fail(NS_ERR_UNSUPPORTED, "the batched entry runs the FP64 and Ozaki paths only");
  if (batch < 1 || batch > 65535) return fail(NS_ERR_INVALID_ARG, "batch must be in [1, 65535]");
  if (!H || !R || !ws || !outs || !s || !alpha || !k) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (stride_h < d * d || stride_r < d * d) return fail(NS_ERR_INVALID_ARG, "strides must be >= d*d");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  std::vector<JobParams> jobs(batch);
  bool any_auto = false;
  for (int64_t b = 0; b < batch; ++b) {
    if (!std::isfinite(s[b])) return fail(NS_ERR_INVALID_ARG, "s[%lld] not finite", (long long)b);
    if (!(alpha[b] >= 0.0) || !std::isfinite(alpha[b]))
      return fail(NS_ERR_INVALID_ARG, "alpha[%lld] must be finite and > 0 (or 0: device Gershgorin bound)", (long long)b);
    if (k[b] < 0 || k[b] > d) return fail(NS_ERR_INVALID_ARG, "k[%lld] out of [0, d]", (long long)b);
    jobs[b] = JobParams{s[b], alpha[b], k[b], 0};
    any_auto |= alpha[b] == 0.0;
  }
  const bool ozaki = (prec == NS_PREC_FP64_OZAKI);
  const Layout L = make_layout(d, batch, false, ozaki);
  if (ws_bytes < L.total)
    return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  if (any_auto) {   // N1: per-job ||H_b - s_b I||_inf on the device (job b's Y buffer is scratch), one readback
    cudaStream_t cs = static_cast<cudaStream_t>(stream);
    double* Yb = reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + L.off_y);
    const size_t js = (size_t)L.d_pad * L.d_pad;
    std::vector<double> a(batch, 0.0);
    for (int64_t b = 0; b < batch; ++b)
      if (jobs[b].alpha == 0.0) {
        NS_CUDA(launch_scale_bound(H + b * stride_h, d, (int)d, jobs[b].s, Yb + b * js, Yb + b * js + d, cs));
        NS_CUDA(cudaMemcpyAsync(&a[b], Yb + b * js + d, sizeof(double), cudaMemcpyDeviceToHost, cs));
      }
    NS_CUDA(cudaStreamSynchronize(cs));
    for (int64_t b = 0; b < batch; ++b)
      if (jobs[b].alpha == 0.0) {
        if (!std::isfinite(a[b])) return fail(NS_ERR_INVALID_ARG, "H[%lld] - s I has a non-finite entry", (long long)b);
        jobs[b].alpha = a[b] > 0.0 ? a[b] : 1.0;
      }
  }
  std::vector<DevState> states;
  int nl = 0;
  if (ozaki) {
    st = run_ozaki_batch(L, static_cast<uint8_t*>(ws), H, d, stride_h, jobs, max_steps, tol, tm, R, d, stride_r,
                         static_cast<cudaStream_t>(stream), Opts{}, states, &nl);
    xprof_flush();
  } else
    st = run_loop(L, static_cast<uint8_t*>(ws), H, d, stride_h, jobs, max_steps, tol, tm, R, d, stride_r,
                  static_cast<cudaStream_t>(stream), states, &nl);
  if (st != NS_OK) return st;
  for (int64_t b = 0; b < batch; ++b) {
    fill_result(states[b], nl, &outs[b]);
    outs[b].alpha = jobs[b].alpha;
  }
  return NS_OK;
}

ns_status_t ns_reflector_batched_dev(const double* H, int64_t d, int64_t batch, int64_t stride_h, const double* s_dev,
                                     const double* alpha_dev, const int32_t* k_dev, int32_t max_steps, double tol,
                                     ns_tolmode_t tm, ns_precision_t prec, double* R, int64_t stride_r, void* ws,
                                     size_t ws_bytes, void* stream, ns_result_t* outs) {
  g_last_error.clear();
  if (batch < 1 || batch > 65535) return fail(NS_ERR_INVALID_ARG, "batch must be in [1, 65535]");
  if (!s_dev || !alpha_dev || !k_dev) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  // the per-problem scalars are validated on the host before any launch (same contract as the host-array
  // entry): one small copy of 20 bytes per problem and one synchronisation
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  std::vector<double> s(batch), a(batch);
  std::vector<int32_t> k(batch);
  NS_CUDA(cudaMemcpyAsync(s.data(), s_dev, sizeof(double) * batch, cudaMemcpyDeviceToHost, cs));
  NS_CUDA(cudaMemcpyAsync(a.data(), alpha_dev, sizeof(double) * batch, cudaMemcpyDeviceToHost, cs));
  NS_CUDA(cudaMemcpyAsync(k.data(), k_dev, sizeof(int32_t) * batch, cudaMemcpyDeviceToHost, cs));
  NS_CUDA(cudaStreamSynchronize(cs));
  return ns_reflector_batched(H, d, batch, stride_h, s.data(), a.data(), k.data(), max_steps, tol, tm, prec, R,
                              stride_r, ws, ws_bytes, stream, outs);
}

size_t ns_workspace_bytes_inertia(int64_t d, ns_precision_t prec) {
  if (d < 1) return 0;
  return align256(ns_workspace_bytes(d, prec)) + align256(sizeof(double) * (size_t)d * (size_t)d);
}

// Inertia probe (N1; alg:ssr step 3 "estimate the target-gap endpoints", realised with the trace
// certificate of prop:exact): #{i : lambda_i(H) < s} = round((d - tr X_m)/2) for the NS iterate X_m of
// X_0 = (H - sI)/alpha, alpha = ||H - sI||_inf >= ||H - sI||_2 (so spec(X_0) c [-1, 1]), run until
// ||X_m^2 - I||_F < 1/(2 sqrt d).  Then every |x_i| <= 1 has the sign of lambda_i - s (lem:NSsign) and
// sum_i (1 - |x_i|) <= sum_i (1 - x_i^2) <= sqrt(d) ||X_m^2 - I||_F < 1/2, so (d - tr X_m)/2 is within 1/4
// of the number of negative x_i: the rounded certificate IS the count.
ns_status_t ns_inertia(const double* H, int64_t d, int64_t ldh, double s, ns_precision_t prec, int32_t max_steps,
                       void* ws, size_t ws_bytes, void* stream, int64_t* count, int32_t* resolved, ns_result_t* out) {
  g_last_error.clear();
  if (!count || !resolved || !out || !ws || !H) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (prec != NS_PREC_FP64 && prec != NS_PREC_FP64_OZAKI)
    return fail(NS_ERR_UNSUPPORTED, "inertia probes run on the FP64 or Ozaki path");
  if (d < 1 || d > 65536) return fail(NS_ERR_INVALID_ARG, "d must be in [1, 65536]");
  if (ws_bytes < ns_workspace_bytes_inertia(d, prec)) return fail(NS_ERR_WORKSPACE, "workspace too small");
  const size_t base = align256(ns_workspace_bytes(d, prec));
  double* Rs = reinterpret_cast<double*>(static_cast<uint8_t*>(ws) + base);
  const double tol = 0.5 / std::sqrt((double)d);
  ns_status_t st = ns_reflector_ex(H, d, ldh, s, 0.0, 0, max_steps, tol, NS_TOL_ABS, prec, Rs, d, ws, base, stream,
                                   nullptr, out);
  if (st != NS_OK) return st;
  *resolved = (out->flags & NS_F_CONVERGED) && !(out->flags & NS_F_NONFINITE) ? 1 : 0;
  *count = out->index_cert;
  return NS_OK;
}

// Endpoint bisection with inertia probes (N1): brackets lambda_k in (a_k, b_k] and lambda_{k+1} in
// (a_k1, b_k1] (count(a) <= k-1 < k <= count(b), and likewise for k+1), refining the wider bracket at its
// midpoint, until the estimated midpoint is certified admissible by prop:reuse_refresh (half the estimated
// gap exceeds the estimate error eps) with eps <= rel_eps * estimated gap.  The reference algorithm (same
// probe sequence, same floating-point formulas) is oracle/setup.py shift_bisect.
ns_status_t ns_shift_bisect(const double* H, int64_t d, int64_t ldh, int32_t k, double lo, double hi, double rel_eps,
                            int32_t max_probes, ns_precision_t prec, void* ws, size_t ws_bytes, void* stream,
                            ns_bisect_t* out) {
  g_last_error.clear();
  if (!out || !ws || !H) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (d < 2 || d > 65536) return fail(NS_ERR_INVALID_ARG, "d must be in [2, 65536]");
  if (k < 1 || k > d - 1) return fail(NS_ERR_INVALID_ARG, "k must lie in [1, d - 1] (the gap (lambda_k, lambda_k+1))");
  if (!(rel_eps > 0.0) || !(rel_eps < 0.5)) return fail(NS_ERR_INVALID_ARG, "rel_eps must lie in (0, 0.5)");
  if (max_probes < 1) return fail(NS_ERR_INVALID_ARG, "max_probes must be >= 1");
  if (ws_bytes < ns_workspace_bytes_inertia(d, prec)) return fail(NS_ERR_WORKSPACE, "workspace too small");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  *out = ns_bisect_t{};
  if (!(lo < hi) || !std::isfinite(lo) || !std::isfinite(hi)) {
    // default bracket: [-||H||_inf, ||H||_inf] contains the spectrum (count = 0 / d at the ends, not probed)
    double nrm = 0.0;
    ns_status_t st = device_scale_bound(H, ldh, (int)d, 0.0, static_cast<double*>(ws), cs, &nrm);
    if (st != NS_OK) return st;
    hi = nrm * (1.0 + 1e-12) + 1e-300;
    lo = -hi;
  }
  double ak = lo, bk = hi, ak1 = lo, bk1 = hi;
  int probes = 0, unresolved = 0;
  ns_result_t r{};
  for (;;) {
    const double lk = 0.5 * (ak + bk), lk1 = 0.5 * (ak1 + bk1);
    const double eps = 0.5 * std::max(bk - ak, bk1 - ak1);
    const double gap = lk1 - lk;
    if (gap > 0.0 && 0.5 * gap > eps && eps <= rel_eps * gap) {
      out->ok = 1;
      break;
    }
    if (probes >= max_probes) break;
    const bool refine_k = (bk - ak) >= (bk1 - ak1);
    const double a = refine_k ? ak : ak1, b = refine_k ? bk : bk1;
    double sp = 0.5 * (a + b);
    int64_t c = 0;
    int32_t res = 0;
    for (int tries = 0; tries < 8; ++tries) {
      ns_status_t st = ns_inertia(H, d, ldh, sp, prec, 100, ws, ws_bytes, stream, &c, &res, &r);
      if (st != NS_OK) return st;
      ++probes;
      if (res) break;
      ++unresolved;                                // s on (or within ~1e-17 of) an eigenvalue: nudge
      sp = sp + (b - a) * std::ldexp(1.0, -20 + tries);
    }
    if (!res) return fail(NS_ERR_CUDA, "inertia probe unresolved after 8 nudges at s = %.17g", sp);
    if (c <= k - 1) {
      ak = std::max(ak, sp);
      ak1 = std::max(ak1, sp);
    } else if (c == k) {
      bk = std::min(bk, sp);
      ak1 = std::max(ak1, sp);
    } else {
      bk = std::min(bk, sp);
      bk1 = std::min(bk1, sp);
    }
  }
  out->lam_k_lo = ak;
  out->lam_k_hi = bk;
  out->lam_k1_lo = ak1;
  out->lam_k1_hi = bk1;
  out->eps = 0.5 * std::max(bk - ak, bk1 - ak1);
  out->s = 0.5 * (0.5 * (ak + bk) + 0.5 * (ak1 + bk1));
  out->probes = probes;
  out->unresolved = unresolved;
  if (out->ok) {   // the scale at the returned shift (device Gershgorin bound)
    double al = 0.0;
    ns_status_t st = device_scale_bound(H, ldh, (int)d, out->s, static_cast<double*>(ws), cs, &al);
    if (st != NS_OK) return st;
    out->alpha = al;
  }
  return NS_OK;
}

int ns_debug_small_trace(unsigned long long* out, int n) { return small_trace_read(out, n); }
int ns_debug_p64_trace(void* device_buffer, unsigned long long capacity) {
  return p64_trace_set(static_cast<unsigned long long*>(device_buffer), capacity);
}

void ns_debug_mx_trace(void* device_buffer) { g_mx_trace = static_cast<unsigned long long*>(device_buffer); }

ns_status_t ns_symm_product(const double* A, const double* B, double* C, int64_t d, int64_t ld, int32_t mode,
                            ns_precision_t prec, void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (d < 1 || d > 65536) return fail(NS_ERR_INVALID_ARG, "bad d");
  if (ld < d) return fail(NS_ERR_INVALID_ARG, "ld must be >= d");
  if (mode < 0 || mode > 2) return fail(NS_ERR_INVALID_ARG, "mode must be 0, 1 or 2");
  if (prec != NS_PREC_FP64 && prec != NS_PREC_MIXED_BF16X3 && prec != NS_PREC_MIXED_TF32X3 &&
      prec != NS_PREC_FP64_OZAKI)
    return fail(NS_ERR_UNSUPPORTED, "precision not available");
  if (prec == NS_PREC_FP64_OZAKI && d > kOzMaxD) return fail(NS_ERR_UNSUPPORTED, "Ozaki products need d <= %d", kOzMaxD);
  if (!A || !B || !C || !ws) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const bool tf32 = (prec == NS_PREC_MIXED_TF32X3);
  const bool mixed = (prec == NS_PREC_MIXED_BF16X3) || tf32;
  const bool ozaki = (prec == NS_PREC_FP64_OZAKI);
  const Layout L = make_layout(d, 1, mixed, ozaki || mixed, tf32);
  if (ws_bytes < L.total) return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  double* Pa = reinterpret_cast<double*>(w + L.off_xa);   // padded A
  double* Pb = reinterpret_cast<double*>(w + L.off_xb);   // padded B
  double* Pc = reinterpret_cast<double*>(w + L.off_y);    // padded C
  int2* tiles = reinterpret_cast<int2*>(w + (mode == 2 ? L.off_full : L.off_tiles));
  JobParams* djobs = reinterpret_cast<JobParams*>(w + L.off_jobs);
  std::vector<int2> tl = (mode == 2) ? make_tiles_full(L.n) : make_tiles(L.n);
  NS_CUDA(cudaMemcpyAsync(tiles, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, cs));
  JobParams unit{0.0, 1.0, 0, 0};
  NS_CUDA(cudaMemcpyAsync(djobs, &unit, sizeof(unit), cudaMemcpyHostToDevice, cs));
  // pad (and symmetrise from the upper triangle, s = 0, alpha = 1)
  NS_CUDA(launch_init(A, ld, 0, Pa, djobs, L.d, L.d_pad, 1, cs));
  NS_CUDA(launch_init(B, ld, 0, Pb, djobs, L.d, L.d_pad, 1, cs));
  double* partial = reinterpret_cast<double*>(w + (mode == 0 ? L.off_res : L.off_tr));
  ns_status_t s;
  if (ozaki) {
    int8_t* slA = reinterpret_cast<int8_t*>(w + L.off_ozx);
    int8_t* slB = reinterpret_cast<int8_t*>(w + L.off_ozy);
    int* eA = reinterpret_cast<int*>(w + L.off_oex);
    int* eB = reinterpret_cast<int*>(w + L.off_oey);
    int2* otiles = reinterpret_cast<int2*>(w + L.off_otiles);
    std::vector<int2> ot = oz_tile_list(L.n, mode != 2);
    NS_CUDA(cudaMemcpyAsync(otiles, ot.data(), ot.size() * sizeof(int2), cudaMemcpyHostToDevice, cs));
    NS_CUDA(launch_ozaki_slice(Pa, slA, eA, L.d_pad, 1, cs));
    NS_CUDA(launch_ozaki_slice(Pb, slB, eB, L.d_pad, 1, cs));
    CUtensorMap tA, tB;
    if ((s = encode_map_i8(&tA, slA, L.d_pad, kOzSlices, kTile)) != NS_OK) return s;
    if ((s = encode_map_i8(&tB, slB, L.d_pad, kOzSlices, 64)) != NS_OK) return s;
    double* opart = reinterpret_cast<double*>(w + (mode == 0 ? L.off_ores : L.off_otr));
    OzParams p{otiles, (int)ot.size(), L.d_pad / 64, L.d, L.d_pad, 0, Pc, Pa, eA, eB, opart, nullptr, mode};
    NS_CUDA(oz_product(tA, tB, p, 1, cs));
  } else if (!mixed) {
    CUtensorMap tA, tB;
    if ((s = encode_map(&tA, Pa, L.d_pad, 1)) != NS_OK) return s;
    if ((s = encode_map(&tB, Pb, L.d_pad, 1)) != NS_OK) return s;
    ProdParams p{tiles, (int)tl.size(), L.d_pad / kBK, L.d, L.d_pad, 0, Pc, Pa, partial, nullptr, mode};
    NS_CUDA(launch_product(tA, tB, p, 1, cs));
  } else {
    void* planesA = w + L.off_px;
    void* planesB = w + L.off_py;
    NS_CUDA(launch_split_planes(Pa, planesA, L.d_pad, 1, cs, tf32));
    NS_CUDA(launch_split_planes(Pb, planesB, L.d_pad, 1, cs, tf32));
    CUtensorMap tA, tB;
    const bool mx2 = use_mx2() && !tf32;
    if ((s = encode_map_bf16(&tA, planesA, L.d_pad, 2, tf32)) != NS_OK) return s;
    if ((s = encode_map_bf16(&tB, planesB, L.d_pad, 2, tf32, mx2 ? 64 : kTile)) != NS_OK) return s;
    int nt = (int)tl.size();
    if (mx2) {
      const std::vector<int2> pl = make_tiles_pairs(L.n, mode != 2);
      NS_CUDA(cudaMemcpyAsync(tiles, pl.data(), pl.size() * sizeof(int2), cudaMemcpyHostToDevice, cs));
      nt = 2 * (int)pl.size();
    }
    MxParams p{tiles, nt, L.d_pad / (tf32 ? 32 : kMxBK), L.d, L.d_pad, 0, Pc, Pa, nullptr, partial,
               nullptr, mode, tf32 ? 1 : 0};
    p.trace = g_mx_trace;                  // diagnostics only (ns_debug_mx_trace)
    NS_CUDA(mx2 ? launch_mx2_product(tA, tB, p, 1, cs) : launch_mx_product(tA, tB, p, 1, cs));
  }
  NS_CUDA(cudaMemcpy2DAsync(C, (size_t)ld * 8, Pc, (size_t)L.d_pad * 8, (size_t)d * 8, (size_t)d,
                            cudaMemcpyDeviceToDevice, cs));
  NS_CUDA(cudaStreamSynchronize(cs));
  return NS_OK;
}

struct ns_comm {
  ncclComm_t comm;
  int rank;
  int nranks;
  CommCtx ctx;
};

ns_status_t ns_comm_get_unique_id(uint8_t id[128]) {
  g_last_error.clear();
  if (!id) return fail(NS_ERR_INVALID_ARG, "null id");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
  ncclUniqueId u;
  NS_NCCL(ncclGetUniqueId(&u));
  memcpy(id, &u, 128);
  return NS_OK;
}

ns_status_t ns_comm_init(int rank, int nranks, const uint8_t id[128], ns_comm_t** comm) {
  g_last_error.clear();
  if (!id || !comm) return fail(NS_ERR_INVALID_ARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NS_ERR_INVALID_ARG, "bad rank/nranks");
  ncclUniqueId u;
  memcpy(&u, id, 128);
  ns_comm_t* c = new ns_comm_t{nullptr, rank, nranks, CommCtx{}};
  ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(NS_ERR_NCCL, "ncclCommInitRank failed: %s", ncclGetErrorString(r));
  }
  c->ctx.comm = c->comm;
  c->ctx.rank = rank;
  c->ctx.nranks = nranks;
  if (cudaStreamCreateWithFlags(&c->ctx.cst, cudaStreamNonBlocking) != cudaSuccess) {
    ncclCommDestroy(c->comm);
    delete c;
    return fail(NS_ERR_CUDA, "communication stream creation failed");
  }
  *comm = c;
  return NS_OK;
}

ns_status_t ns_comm_init_host(int rank, int nranks, ns_host_allgather_fn allgather, void* user, ns_comm_t** comm) {
  g_last_error.clear();
  if (!allgather || !comm) return fail(NS_ERR_INVALID_ARG, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NS_ERR_INVALID_ARG, "bad rank/nranks");
  ns_comm_t* c = new ns_comm_t{nullptr, rank, nranks, CommCtx{}};
  c->ctx.host_fn = allgather;
  c->ctx.host_user = user;
  c->ctx.rank = rank;
  c->ctx.nranks = nranks;
  if (cudaStreamCreateWithFlags(&c->ctx.cst, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return fail(NS_ERR_CUDA, "communication stream creation failed");
  }
  *comm = c;
  return NS_OK;
}

ns_status_t ns_comm_destroy(ns_comm_t* comm) {
  g_last_error.clear();
  if (!comm) return NS_OK;
  close_peers(comm->ctx);
  for (cudaEvent_t e : comm->ctx.ev) cudaEventDestroy(e);
  if (comm->ctx.cst) cudaStreamDestroy(comm->ctx.cst);
  ncclResult_t r = comm->comm ? ncclCommDestroy(comm->comm) : ncclSuccess;
  delete comm;
  if (r != ncclSuccess) return fail(NS_ERR_NCCL, "ncclCommDestroy failed: %s", ncclGetErrorString(r));
  return NS_OK;
}

ns_status_t ns_symm_product_shard(const double* A, const double* B, double* const* C_list, int32_t n_dst, int64_t d,
                                  int32_t mode, int32_t rank, int32_t nranks, void* ws, size_t ws_bytes, void* stream) {
  g_last_error.clear();
  if (d < kTile || d > 65536 || d % kTile != 0) return fail(NS_ERR_INVALID_ARG, "d must be a multiple of 128 in [128, 65536]");
  if (mode < 0 || mode > 1) return fail(NS_ERR_INVALID_ARG, "mode must be 0 or 1");
  if (nranks < 1 || rank < 0 || rank >= nranks || n_dst < 1 || n_dst > 64)
    return fail(NS_ERR_INVALID_ARG, "bad rank / nranks / n_dst");
  if (!A || !B || !C_list || !ws) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  for (int q = 0; q < n_dst; ++q)
    if (!C_list[q]) return fail(NS_ERR_INVALID_ARG, "null destination");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const Layout L = make_layout(d, 1, false);
  if (ws_bytes < L.total) return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, L.total);
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  uint8_t* w = static_cast<uint8_t*>(ws);
  int2* tiles = reinterpret_cast<int2*>(w + L.off_tiles);
  double** dst = reinterpret_cast<double**>(w + L.off_full);                 // n_dst C bases, n_dst partial bases
  double* part = reinterpret_cast<double*>(w + L.off_res);
  const std::vector<int2> mt = shard_tiles(make_tiles(L.n), nranks, rank);
  if (mt.empty()) return NS_OK;
  std::vector<double*> h(2 * (size_t)n_dst);
  for (int q = 0; q < n_dst; ++q) {
    h[q] = C_list[q];
    h[n_dst + q] = part;
  }
  NS_CUDA(cudaMemcpyAsync(tiles, mt.data(), mt.size() * sizeof(int2), cudaMemcpyHostToDevice, cs));
  NS_CUDA(cudaMemcpyAsync(dst, h.data(), h.size() * sizeof(double*), cudaMemcpyHostToDevice, cs));
  CUtensorMap tA, tB;
  ns_status_t s;
  if ((s = encode_map(&tA, A, L.d_pad, 1)) != NS_OK) return s;
  if ((s = encode_map(&tB, B, L.d_pad, 1)) != NS_OK) return s;
  ProdParams pp{tiles, (int)mt.size(), L.d_pad / kBK, L.d, L.d_pad, 0, C_list[0], A, part, nullptr, mode};
  pp.dst = dst;
  pp.dst_part = dst + n_dst;
  pp.n_dst = n_dst;
  pp.gt_off = rank;
  pp.gt_stride = nranks;
  pp.n_tiles_total = L.n_tiles;
  NS_CUDA(launch_product(tA, tB, pp, 1, cs));
  NS_CUDA(cudaStreamSynchronize(cs));
  return NS_OK;
}

size_t ns_workspace_bytes_sharded_emulated(int64_t d, int nranks) {
  if (d < 1 || nranks < 1) return 0;
  return align256(make_shard_layout(d, nranks, 0).total) * (size_t)nranks;
}

ns_status_t ns_reflector_sharded_emulated(int32_t nranks, const double* H, int64_t d, int64_t ldh, double s,
                                          double alpha, int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm,
                                          double* R, int64_t ldr, void* ws, size_t ws_bytes, void* stream,
                                          int32_t flags, ns_result_t* out) {
  g_last_error.clear();
  ns_status_t st = check_common(d, max_steps, tol, tm, NS_PREC_FP64);
  if (st != NS_OK) return st;
  if (nranks < 1 || nranks > 64) return fail(NS_ERR_INVALID_ARG, "nranks must be in [1, 64]");
  if (flags & ~3) return fail(NS_ERR_INVALID_ARG, "flags: bit 0 = block-row input, bit 1 = sender mirror");
  if (!H || !R || !ws || !out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (ldh < d || ldr < d) return fail(NS_ERR_INVALID_ARG, "leading dimensions must be >= d");
  if (!std::isfinite(s)) return fail(NS_ERR_INVALID_ARG, "shift s must be finite");
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return fail(NS_ERR_INVALID_ARG, "alpha must be finite and > 0");
  if (k < 0 || k > d) return fail(NS_ERR_INVALID_ARG, "k must lie in [0, d]");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const size_t stride = align256(make_shard_layout(d, nranks, 0).total);
  if (ws_bytes < stride * (size_t)nranks)
    return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, stride * (size_t)nranks);
  DevState ds;
  int nl = 0;
  st = run_sharded_emulated(d, nranks, static_cast<uint8_t*>(ws), stride, H, ldh, JobParams{s, alpha, k, 0},
                            max_steps, tol, tm, R, ldr, static_cast<cudaStream_t>(stream), ds, &nl, flags);
  if (st != NS_OK) return st;
  fill_result(ds, nl, out);
  out->alpha = alpha;
  return NS_OK;
}

ns_status_t ns_shard_plan(int64_t d, int nranks, int rank, int32_t* tiles_ij, int32_t cap, int32_t* n_out) {
  g_last_error.clear();
  if (d < 1 || d > 65536 || nranks < 1 || rank < 0 || rank >= nranks || !n_out)
    return fail(NS_ERR_INVALID_ARG, "bad arguments");
  const Layout L = make_layout(d, 1, false);
  std::vector<int2> mt = shard_tiles(make_tiles(L.n), nranks, rank);
  *n_out = (int32_t)mt.size();
  for (int32_t i = 0; i < (int32_t)mt.size() && i < cap && tiles_ij; ++i) {
    tiles_ij[2 * i] = mt[i].x;
    tiles_ij[2 * i + 1] = mt[i].y;
  }
  return NS_OK;
}

ns_status_t ns_shard_chunks(int64_t d, int nranks, int32_t* n_chunks, int32_t* chunk_slots) {
  g_last_error.clear();
  if (d < 1 || d > 65536 || nranks < 1 || !n_chunks || !chunk_slots) return fail(NS_ERR_INVALID_ARG, "bad arguments");
  const ShardLayout SL = make_shard_layout(d, nranks, 0);
  *n_chunks = SL.n_chunks;
  *chunk_slots = SL.cs;
  return NS_OK;
}

size_t ns_workspace_bytes_sharded(int64_t d, int nranks) {
  if (d < 1 || nranks < 1) return 0;
  return make_shard_layout(d, nranks, 0).total;
}

ns_status_t ns_reflector_sharded(ns_comm_t* comm, const double* H, int64_t d, int64_t ldh, double s, double alpha,
                                 int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm, double* R, int64_t ldr,
                                 void* ws, size_t ws_bytes, void* stream, ns_result_t* out) {
  g_last_error.clear();
  if (!comm) return fail(NS_ERR_INVALID_ARG, "null communicator");
  ns_status_t st = check_common(d, max_steps, tol, tm, NS_PREC_FP64);
  if (st != NS_OK) return st;
  if (!H || !R || !ws || !out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (ldh < d || ldr < d) return fail(NS_ERR_INVALID_ARG, "leading dimensions must be >= d");
  if (!std::isfinite(s)) return fail(NS_ERR_INVALID_ARG, "shift s must be finite");
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return fail(NS_ERR_INVALID_ARG, "alpha must be finite and > 0");
  if (k < 0 || k > d) return fail(NS_ERR_INVALID_ARG, "k must lie in [0, d]");
  if (R == H) return fail(NS_ERR_INVALID_ARG, "R must not alias H");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const ShardLayout SL = make_shard_layout(d, comm->nranks, comm->rank);
  if (ws_bytes < SL.total)
    return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, SL.total);
  DevState ds;
  int nl = 0;
  st = run_sharded(comm->ctx, SL, static_cast<uint8_t*>(ws), H, nullptr, ldh, 0, d, JobParams{s, alpha, k, 0},
                   max_steps, tol, tm, R, ldr, static_cast<cudaStream_t>(stream), ds, &nl, shard_sender_mirror());
  if (st != NS_OK) return st;
  fill_result(ds, nl, out);
  out->alpha = alpha;
  return NS_OK;
}

ns_status_t ns_shard_rows(int64_t d, int nranks, int rank, int64_t* row0, int64_t* row1) {
  g_last_error.clear();
  if (d < 1 || nranks < 1 || rank < 0 || rank >= nranks || !row0 || !row1)
    return fail(NS_ERR_INVALID_ARG, "bad arguments");
  if (d % nranks != 0) return fail(NS_ERR_INVALID_ARG, "d = %lld is not divisible by nranks = %d", (long long)d, nranks);
  *row0 = d / nranks * rank;
  *row1 = d / nranks * (rank + 1);
  return NS_OK;
}

ns_status_t ns_reflector_sharded_rows(ns_comm_t* comm, const double* H_rows, int64_t d, int64_t ldh, double s,
                                      double alpha, int32_t k, int32_t max_steps, double tol, ns_tolmode_t tm,
                                      ns_precision_t prec, double* R_rows, int64_t ldr, void* ws, size_t ws_bytes,
                                      void* stream, ns_result_t* out) {
  g_last_error.clear();
  if (!comm) return fail(NS_ERR_INVALID_ARG, "null communicator");
  ns_status_t st = check_common(d, max_steps, tol, tm, prec);
  if (st != NS_OK) return st;
  if (prec != NS_PREC_FP64)
    return fail(NS_ERR_UNSUPPORTED, "the sharded path runs FP64 DMMA products only (prec = %d)", (int)prec);
  if (d % comm->nranks != 0)
    return fail(NS_ERR_INVALID_ARG, "d = %lld is not divisible by nranks = %d", (long long)d, comm->nranks);
  const long long rows = d / comm->nranks, r0 = rows * comm->rank, r1 = r0 + rows;
  if ((!H_rows || !R_rows) && rows > 0) return fail(NS_ERR_INVALID_ARG, "null H_rows / R_rows");
  if (!ws || !out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (ldh < d || ldr < d) return fail(NS_ERR_INVALID_ARG, "leading dimensions must be >= d");
  if (!std::isfinite(s)) return fail(NS_ERR_INVALID_ARG, "shift s must be finite");
  if (!(alpha > 0.0) || !std::isfinite(alpha)) return fail(NS_ERR_INVALID_ARG, "alpha must be finite and > 0");
  if (k < 0 || k > d) return fail(NS_ERR_INVALID_ARG, "k must lie in [0, d]");
  if (R_rows == H_rows) return fail(NS_ERR_INVALID_ARG, "R_rows must not alias H_rows");
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  const ShardLayout SL = make_shard_layout(d, comm->nranks, comm->rank);
  if (ws_bytes < SL.total)
    return fail(NS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, SL.total);
  DevState ds;
  int nl = 0;
  st = run_sharded(comm->ctx, SL, static_cast<uint8_t*>(ws), nullptr, H_rows, ldh, r0, r1, JobParams{s, alpha, k, 0},
                   max_steps, tol, tm, R_rows, ldr, static_cast<cudaStream_t>(stream), ds, &nl, shard_sender_mirror());
  if (st != NS_OK) return st;
  fill_result(ds, nl, out);
  out->alpha = alpha;
  return NS_OK;
}

size_t ns_workspace_bytes_setup(int64_t d) { return d < 1 ? 0 : align256(sizeof(double) * (size_t)(d + 1)); }

ns_status_t ns_scale_bound(const double* H, int64_t d, int64_t ldh, double s, void* ws, size_t ws_bytes,
                           void* stream, double* alpha_out) {
  g_last_error.clear();
  if (!H || !ws || !alpha_out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (d < 1 || d > 65536 || ldh < d) return fail(NS_ERR_INVALID_ARG, "bad d / ldh");
  if (!std::isfinite(s)) return fail(NS_ERR_INVALID_ARG, "shift must be finite");
  if (ws_bytes < ns_workspace_bytes_setup(d)) return fail(NS_ERR_WORKSPACE, "workspace too small");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  double* part = static_cast<double*>(ws);
  double* dout = part + d;
  NS_CUDA(launch_scale_bound(H, ldh, (int)d, s, part, dout, cs));
  NS_CUDA(cudaMemcpyAsync(alpha_out, dout, sizeof(double), cudaMemcpyDeviceToHost, cs));
  NS_CUDA(cudaStreamSynchronize(cs));
  if (!std::isfinite(*alpha_out)) return fail(NS_ERR_INVALID_ARG, "H - sI has a non-finite entry: no scale bound");
  return NS_OK;
}

ns_status_t ns_shift_certificate(double lam_k_hat, double lam_k1_hat, double eps, double s, double delta,
                                 ns_shift_cert_t* out) {
  g_last_error.clear();
  if (!out) return fail(NS_ERR_INVALID_ARG, "null output");
  if (!std::isfinite(lam_k_hat) || !std::isfinite(lam_k1_hat) || !std::isfinite(s) || !(eps >= 0.0) ||
      !(delta >= 0.0) || !std::isfinite(eps) || !std::isfinite(delta))
    return fail(NS_ERR_INVALID_ARG, "estimates must be finite, eps and delta >= 0");
  ns_shift_cert_t c{};
  c.margin_hat = std::min(s - lam_k_hat, lam_k1_hat - s);
  c.admissible = c.margin_hat > eps ? 1 : 0;
  c.margin_lb = c.margin_hat - eps;
  c.reuse_ok = (c.admissible && delta < c.margin_hat - eps) ? 1 : 0;
  c.reuse_margin_lb = c.margin_hat - eps - delta;
  c.midpoint = 0.5 * (lam_k_hat + lam_k1_hat);
  c.midpoint_ok = (0.5 * (lam_k1_hat - lam_k_hat) > eps) ? 1 : 0;
  *out = c;
  return NS_OK;
}

size_t ns_workspace_bytes_alg1(int32_t nruns) {
  if (nruns < 1) return 0;
  return align256(sizeof(int) * (size_t)nruns) + align256(sizeof(OuterResult) * (size_t)nruns);
}

ns_status_t ns_alg1_rotated_quartic_ex(const double* Q, int64_t d, int32_t nruns, const int32_t* k,
                                       const double* x0, int32_t m, double eta, int32_t max_iters, double grad_tol,
                                       const ns_alg1_policy_t* pol, double* x_out, void* ws, size_t ws_bytes,
                                       void* stream, ns_alg1_result_t* out) {
  g_last_error.clear();
  if (!Q || !k || !x0 || !x_out || !ws || !out) return fail(NS_ERR_INVALID_ARG, "null pointer argument");
  if (d < 2 || d > 64) return fail(NS_ERR_INVALID_ARG, "d must lie in [2, 64] (one CTA per run)");
  if (nruns < 1 || nruns > 1 << 20) return fail(NS_ERR_INVALID_ARG, "bad nruns");
  if (m < 0 || m > 64 || max_iters < 0) return fail(NS_ERR_INVALID_ARG, "bad depth / iteration budget");
  if (!(eta > 0.0) || !std::isfinite(eta) || !(grad_tol >= 0.0)) return fail(NS_ERR_INVALID_ARG, "bad eta / grad_tol");
  ns_alg1_policy_t pp{NS_SHIFT_MIDPOINT, 0, 0.5, 0.25, 0.0, 0.0};
  if (pol) pp = *pol;
  if (pp.policy < NS_SHIFT_MIDPOINT || pp.policy > NS_SHIFT_REUSE) return fail(NS_ERR_INVALID_ARG, "unknown shift policy");
  if (!(pp.damp >= 0.0 && pp.damp < 1.0)) return fail(NS_ERR_INVALID_ARG, "damp must lie in [0, 1)");
  if (!(pp.clip > 0.0 && pp.clip <= 0.5)) return fail(NS_ERR_INVALID_ARG, "clip must lie in (0, 1/2]");
  if (!(pp.reuse_margin >= 0.0) || !std::isfinite(pp.reuse_margin) || !(pp.eps >= 0.0) || !std::isfinite(pp.eps))
    return fail(NS_ERR_INVALID_ARG, "reuse_margin and eps must be finite and >= 0");
  for (int r = 0; r < nruns; ++r)
    if (k[r] < 1 || k[r] >= d) return fail(NS_ERR_INVALID_ARG, "k[%d] must lie in [1, d-1]", r);
  if ((reinterpret_cast<uintptr_t>(ws) & 255) != 0) return fail(NS_ERR_INVALID_ARG, "workspace must be 256-byte aligned");
  if (ws_bytes < ns_workspace_bytes_alg1(nruns)) return fail(NS_ERR_WORKSPACE, "workspace too small");
  cudaStream_t cs = static_cast<cudaStream_t>(stream);
  int* dk = static_cast<int*>(ws);
  OuterResult* dres = reinterpret_cast<OuterResult*>(static_cast<uint8_t*>(ws) + align256(sizeof(int) * (size_t)nruns));
  NS_CUDA(cudaMemcpyAsync(dk, k, sizeof(int) * nruns, cudaMemcpyHostToDevice, cs));
  OuterParams p{m, max_iters, eta, grad_tol, pp.policy, 0, pp.damp, pp.clip, pp.reuse_margin, pp.eps};
  NS_CUDA(launch_outer(Q, (int)d, dk, x0, p, x_out, dres, nruns, cs));
  std::vector<OuterResult> hr(nruns);
  NS_CUDA(cudaMemcpyAsync(hr.data(), dres, sizeof(OuterResult) * nruns, cudaMemcpyDeviceToHost, cs));
  NS_CUDA(cudaStreamSynchronize(cs));
  for (int r = 0; r < nruns; ++r) {
    out[r].iters = hr[r].iters;
    out[r].morse_index = hr[r].morse_index;
    out[r].success = hr[r].success;
    out[r].stop_reason = hr[r].stop_reason;
    out[r].grad_norm = hr[r].grad_norm;
    out[r].refreshes = hr[r].refreshes;
    out[r].pad = 0;
    out[r].s_last = hr[r].s_last;
  }
  return NS_OK;
}

ns_status_t ns_alg1_rotated_quartic(const double* Q, int64_t d, int32_t nruns, const int32_t* k, const double* x0,
                                    int32_t m, double eta, int32_t max_iters, double grad_tol, double* x_out,
                                    void* ws, size_t ws_bytes, void* stream, ns_alg1_result_t* out) {
  return ns_alg1_rotated_quartic_ex(Q, d, nruns, k, x0, m, eta, max_iters, grad_tol, nullptr, x_out, ws, ws_bytes,
                                    stream, out);
}

void ns_profile_enable(int on) { prof().on = (on != 0); }
void ns_profile_reset(void) { prof().acc = ns_profile_t{}; }
void ns_profile_get(ns_profile_t* out) {
  if (out) *out = prof().acc;
}

const char* ns_build_info(void) {
  return "libnsreflector FP64 DMMA/TMA path; target sm_100a; 128x128 tiles (3 x 64 KB TMA ring, 8 DMMA warps), 64x64 batched tiles, tcgen05 BF16x3 / INT8 Ozaki paths";
}

const char* ns_status_string(ns_status_t st) {
  switch (st) {
    case NS_OK: return "NS_OK";
    case NS_ERR_INVALID_ARG: return "NS_ERR_INVALID_ARG";
    case NS_ERR_CUDA: return "NS_ERR_CUDA";
    case NS_ERR_NCCL: return "NS_ERR_NCCL";
    case NS_ERR_WORKSPACE: return "NS_ERR_WORKSPACE";
    case NS_ERR_UNSUPPORTED: return "NS_ERR_UNSUPPORTED";
  }
  return "NS_ERR_UNKNOWN";
}

const char* ns_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
