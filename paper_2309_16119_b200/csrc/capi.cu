// capi.cu — the C ABI of include/mlra.h: validation with the reference's error
// taxonomy, device upload, workspace, and the kernel sequence of one
// ModuLoRA linear forward / backward.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/mlra.h"
#include <atomic>
#include <chrono>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "qgemm.h"
#include "qgemm_dev.cuh"

using mlra::QWeightDev;

namespace mlra {
static std::atomic<uint64_t> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
// Dev-only host-side profile of the API calls (MLRA_HOSTPROF=1): wall time in
// workspace allocation, tensor-map encoding, kernel launches and whole calls,
// printed to stderr at exit.
struct HostProf {
  std::atomic<uint64_t> ns[5]{}, n[5]{};
  const bool on = getenv("MLRA_HOSTPROF") != nullptr;
  ~HostProf() {
    if (!on) return;
    const char* nm[5] = {"alloc", "tmap", "launch", "call", "free"};
    for (int i = 0; i < 5; ++i)
      fprintf(stderr, "mlra hostprof %-6s %8.2f us total-per-call-avg %llu events\n", nm[i],
              n[3] ? ns[i].load() / 1e3 / n[3].load() : 0.0, (unsigned long long)n[i].load());
  }
};
HostProf g_prof;
struct ProfScope {
  int k;
  std::chrono::steady_clock::time_point t0;
  explicit ProfScope(int kk) : k(kk) {
    if (g_prof.on) t0 = std::chrono::steady_clock::now();
  }
  ~ProfScope() {
    if (!g_prof.on) return;
    g_prof.ns[k] += std::chrono::duration_cast<std::chrono::nanoseconds>(
                        std::chrono::steady_clock::now() - t0).count();
    g_prof.n[k] += 1;
  }
};

HostLaunchTimer::HostLaunchTimer() : impl(g_prof.on ? new ProfScope(2) : nullptr) {}
HostLaunchTimer::~HostLaunchTimer() { delete static_cast<ProfScope*>(impl); }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("MLRA_PDL");
    return e == nullptr || atoi(e) != 0;
  }();
  return on;
}
}  // namespace mlra
using mlra::ProfScope;

struct mlra_qweight {
  QWeightDev d{};
  uint32_t* words = nullptr;
  float2* grid = nullptr;
  uint64_t device_bytes = 0;
  int64_t uncertified = 0;
  // opaque (plugin-owned) formats: every dequantization goes through `hook`
  bool opaque = false;
  mlra_hook hook{};
  std::string hook_name;
  // built-in cb2 plugin state (owned when the qweight came from mlra_cb2_create)
  mlra::Cb2Dev cb2{};
  void* cb2_mem = nullptr;
  // fused cb2 path: the u16 code stream seen as a 2-bit packed matrix + {s, 0} grid
  bool cb2_fused = false;
  QWeightDev cb2_d{};
  float2* cb2_grid = nullptr;
  // built-in lut plugin: the 16-float level table (d.lut points here)
  float* lut_mem = nullptr;
};

namespace {
thread_local std::string g_last_error;
thread_local int g_format_kind = -1;
thread_local uint64_t g_format_offset = 0;
}  // namespace

namespace mlra {
// Error channel shared with the host-side translation units (checkpoint.cpp).
mlra_status set_error(mlra_status st, const std::string& msg) {
  g_last_error = msg;
  g_format_kind = -1;
  g_format_offset = 0;
  return st;
}
mlra_status set_format_error(int kind, uint64_t offset, const std::string& msg) {
  g_last_error = msg;
  g_format_kind = kind;
  g_format_offset = offset;
  return MLRA_ERR_FORMAT;
}
}  // namespace mlra

namespace {

mlra_status fail(mlra_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return st;
}

#define CUDA_TRY(expr)                                                                \
  do {                                                                                \
    cudaError_t e_ = (expr);                                                          \
    if (e_ != cudaSuccess)                                                            \
      return fail(MLRA_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_),     \
                  __FILE__, __LINE__);                                                \
  } while (0)

bool supported_bits(int b) { return b == 2 || b == 3 || b == 4 || b == 8; }
int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

mlra_status check_device() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess)
    return fail(MLRA_ERR_UNSUPPORTED, "no CUDA device: %s", cudaGetErrorString(e));
  int major = 0, minor = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0)
    return fail(MLRA_ERR_UNSUPPORTED, "libmlra is built for sm_100a (B200); device is sm_%d%d",
                major, minor);
  // Per-call workspaces come from the device's stream-ordered pool; keep freed
  // blocks cached instead of returning them to the driver at every sync.
  static bool pool_set[64] = {};
  if (dev < 64 && !pool_set[dev]) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool_set[dev] = true;
  }
  return MLRA_OK;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D tensor [outer x inner] (row stride ld elements). Default: bf16 with a
// SWIZZLE_128B box (tcgen05 operands); the Q ring uses unswizzled u8 / f32.
mlra_status make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer,
                     uint64_t ld, uint32_t box_inner, uint32_t box_outer,
                     CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                     uint32_t esize = 2, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  ProfScope ps(1);
  auto enc = get_encode();
  if (!enc) return fail(MLRA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esize};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(MLRA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): inner=%llu outer=%llu ld=%llu",
                static_cast<int>(r), (unsigned long long)inner, (unsigned long long)outer,
                (unsigned long long)ld);
  return MLRA_OK;
}

// Per-stream workspace arena: one device block reused by every API call on the
// stream (bump allocation; stream order makes reuse safe — a call's side-stream
// work is joined back into the stream before the call returns). A call that
// needs more than the block gets the excess from the stream-ordered pool and
// the block is regrown (stream-ordered free + alloc) for the next call. Calls
// under stream capture, or concurrent calls on one stream, use the pool only.
// (Per-call cudaMallocAsync was ~10 us of host time per buffer, ~11 buffers
// per layer pass: MLRA_HOSTPROF.)
struct Arena {
  char* base = nullptr;
  size_t cap = 0;
  bool busy = false;
};
std::mutex g_arena_mu;
constexpr size_t kArenaMaxItem = size_t{64} << 20;  // bigger buffers (a whole Ŵ, hook slabs): pool
struct ArenaKey {
  int dev;
  cudaStream_t st;
  bool operator==(const ArenaKey& o) const { return dev == o.dev && st == o.st; }
};
struct ArenaKeyHash {
  size_t operator()(const ArenaKey& k) const {
    return std::hash<const void*>()(k.st) * 31u + static_cast<size_t>(k.dev);
  }
};
std::unordered_map<ArenaKey, Arena, ArenaKeyHash>& arenas() {
  static std::unordered_map<ArenaKey, Arena, ArenaKeyHash> m;
  return m;
}

// Stream-ordered scratch owned by one API call.
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;  // pool allocations (freed on the stream at the end)
  Arena* ar = nullptr;
  size_t used = 0, want = 0;
  explicit Scratch(cudaStream_t s) : st(s) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_arena_mu);
    Arena& a = arenas()[ArenaKey{dev, s}];
    if (!a.busy) {
      a.busy = true;
      ar = &a;
    }
  }
  ~Scratch() {
    ProfScope ps(4);
    for (void* p : ptrs) cudaFreeAsync(p, st);
    if (!ar) return;
    if (want > ar->cap) {  // regrow for the next call on this stream
      if (ar->base) cudaFreeAsync(ar->base, st);
      const size_t cap = want + want / 4;
      void* p = nullptr;
      if (cudaMallocAsync(&p, cap, st) == cudaSuccess) {
        ar->base = static_cast<char*>(p);
        ar->cap = cap;
      } else {
        ar->base = nullptr;
        ar->cap = 0;
      }
    }
    std::lock_guard<std::mutex> lk(g_arena_mu);
    ar->busy = false;
  }
  template <typename T>
  T* get(size_t count) {
    ProfScope ps(0);
    const size_t bytes = (count * sizeof(T) + 16 + 255) & ~size_t{255};
    if (ar && bytes <= kArenaMaxItem) {
      want += bytes;
      if (used + bytes <= ar->cap) {
        void* p = ar->base + used;
        used += bytes;
        return static_cast<T*>(p);
      }
    }
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes, st) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

// Activations must be 16-byte aligned rows for TMA and the vectorized skinny
// kernels; otherwise copy into an aligned scratch.
mlra_status aligned_act(Scratch& sc, const void* p, int64_t ld, int64_t m, int64_t cols,
                        const __nv_bfloat16** out, int64_t* out_ld) {
  if (ld % 8 == 0 && reinterpret_cast<uintptr_t>(p) % 16 == 0) {
    *out = static_cast<const __nv_bfloat16*>(p);
    *out_ld = ld;
    return MLRA_OK;
  }
  const int64_t nld = round_up(cols, 8);
  auto* buf = sc.get<__nv_bfloat16>(static_cast<size_t>(m * nld));
  if (!buf) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  CUDA_TRY(cudaMemcpy2DAsync(buf, nld * 2, p, ld * 2, cols * 2, m, cudaMemcpyDeviceToDevice,
                             sc.st));
  *out = buf;
  *out_ld = nld;
  return MLRA_OK;
}

mlra_status check_q(const mlra_qweight* q) {
  if (!q) return fail(MLRA_ERR_CONTRACT, "lp_linear: missing quantized weights");
  return MLRA_OK;
}

// One base GEMM (+ optional LoRA extra K) launch.
struct GemmPlan {
  bool mn;               // false: forward, true: dX
  const __nv_bfloat16* act;
  int64_t ld_act;
  int64_t k_red_valid;   // valid reduction extent of the activations
  const __nv_bfloat16* act_lora = nullptr;   // [m x rp]
  const __nv_bfloat16* w_lora = nullptr;     // [m_total x rp]
  int64_t rp = 0, rank = 0;
  int64_t tokens;
  void* out;
  int64_t ldo;
  bool out_f32;
  const float* bias = nullptr;
  const void* cb2_codebook = nullptr;  // fused cb2 plugin decode (pair kernel, Q ring)
  int e8p = 0;                         // with cb2_codebook: the e8p plugin's decode
  const float* lut = nullptr;          // fused lut plugin decode (pair kernel, Q ring)
  // stream-K / split-K publish flags already zeroed by the pass's prep launch
  // (so no memset node sits between the skinny product and the GEMM, which
  // would break the programmatic launch chain); nullptr: zeroed here
  unsigned* sk_flags_zeroed = nullptr;
  // launch classically: a side stream's kernels (dA/dB) should get the SMs
  // before this GEMM's CTAs, which a programmatic early launch would preempt
  bool no_pdl = false;
};

// One GEMM over the quantized operand described by d. w_mat != nullptr: Ŵ is
// already materialized (bf16 [d.rows x w_ld]) and streamed by TMA; otherwise
// the fused kernel dequantizes d's packed codes tile by tile.
mlra_status run_gemm_d(const QWeightDev& d, const __nv_bfloat16* w_mat, int64_t w_ld,
                       const GemmPlan& gp, Scratch& sc) {
  mlra::GemmMaps maps;
  std::memset(&maps, 0, sizeof(maps));
  mlra::GemmArgs a{};
  a.m_total = gp.mn ? d.cols_pad : d.rows_pad;
  a.m_valid = gp.mn ? d.cols : d.rows;
  a.n_kb_main = static_cast<int>((gp.mn ? d.rows_pad : d.cols_pad) / 64);
  a.n_kb_lora = gp.rank > 0 ? static_cast<int>(gp.rp / 64) : 0;
  if (a.n_kb_lora) {
    const int64_t last = gp.rank - 64 * (a.n_kb_lora - 1);
    a.lora_k16_last = static_cast<int>((last + 15) / 16);
  }
  a.tokens = gp.tokens;
  a.out = gp.out;
  a.ldo = gp.ldo;
  a.bias = gp.bias;
  a.out_pairs = !gp.out_f32 && gp.ldo % 2 == 0 &&
                reinterpret_cast<uintptr_t>(gp.out) % 4 == 0 ? 1 : 0;
  // CTA-pair kernel (512 tokens per tile) or the 1-CTA kernel (256 or 128), by
  // the cost model; MLRA_GEMM=1|2|3 forces the 1-CTA (256) / pair / 1-CTA (128)
  // kernel (tests cover all three).
  a.cb2_codebook = gp.cb2_codebook;
  a.no_pdl = gp.no_pdl ? 1 : 0;
  a.e8p = gp.e8p;
  a.lut = gp.lut;
  int kind = mlra::qgemm_choose(a);
  if (const char* force = getenv("MLRA_GEMM")) kind = atoi(force);
  if (gp.cb2_codebook || gp.lut) kind = 2;  // the plugin decodes live in the pair kernel
  const bool pair = kind == 2;
  a.bn = kind == 3 ? 128 : 256;
  const uint32_t tbox = pair ? 128 : static_cast<uint32_t>(a.bn);
  mlra_status st = make_map(&maps.act, gp.act, gp.k_red_valid, gp.tokens, gp.ld_act, 64, tbox);
  if (st) return st;
  if (a.n_kb_lora) {
    if ((st = make_map(&maps.act_lora, gp.act_lora, gp.rp, gp.tokens, gp.rp, 64, tbox))) return st;
    if ((st = make_map(&maps.w_lora, gp.w_lora, gp.rp, a.m_total, gp.rp, 64, 128))) return st;
  } else {
    maps.act_lora = maps.act;
    maps.w_lora = maps.act;
  }
  const bool w_tma = w_mat != nullptr;
  if (w_tma) {
    if ((st = make_map(&maps.w, w_mat, d.cols, d.rows, w_ld, 64, gp.mn ? 64 : 128))) return st;
  } else {
    maps.w = maps.act;
  }
  maps.codes = maps.act;
  maps.grid = maps.act;
  if (!w_tma && mlra::qgemm_q_tma_ok(d)) {
    // Q ring: 128 codes x 128 weight rows per stage, plus their grid entries
    const int64_t g = d.group;
    const int gfl = 2 * static_cast<int>(g < 128 ? 128 / g : 2);  // floats per row in the box
    a.q_codes_bytes = 128 * 16 * d.bits;
    a.q_grid_bytes = 128 * gfl * 4;
    a.q_stage_bytes = static_cast<int>(round_up(a.q_codes_bytes + a.q_grid_bytes, 128));
    a.q_stages = mlra::qgemm_max_q_stages(
        a.q_stage_bytes,
        gp.cb2_codebook ? (gp.e8p ? mlra::kE8pSmemBytes : mlra::kCb2SmemBytes)
                        : (gp.lut ? mlra::kLutSmemBytes : 0));
    a.q_group_shift = g < 128 ? (g == 32 ? 5 : 6) : -1;
    a.q_group_div128 = g >= 128 ? static_cast<int>(g / 128) : 1;
    {
      const uint64_t d = static_cast<uint64_t>(a.q_group_div128);
      a.q_group_magic = d > 1 ? static_cast<uint32_t>(((1ull << 32) + d - 1) / d) : 0u;
    }
    if (a.q_stages >= 2) {
      if ((st = make_map(&maps.codes, d.words, d.row_words * 4, d.rows_pad, d.row_words * 4,
                         16 * d.bits, 128, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1,
                         CU_TENSOR_MAP_SWIZZLE_NONE)))
        return st;
      if ((st = make_map(&maps.grid, d.grid, 2 * d.ng_pad, d.rows_pad, 2 * d.ng_pad, gfl, 128,
                         CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, CU_TENSOR_MAP_SWIZZLE_NONE)))
        return st;
    } else {
      a.q_stages = 0;
    }
  }
  if (kind == 3 && a.q_stages > 0) {  // the 128-token 1-CTA kernel's deeper ring leaves less room
    const int room = (mlra::qg::SMEM_LIMIT - mlra::qg::qgemm1_smem_fixed(128)) / a.q_stage_bytes;
    a.q_stages = room < 2 ? 0 : (a.q_stages > room ? room : a.q_stages);  // 0: LDG path
  }
  if (const char* tr = getenv("MLRA_TRACE"))  // dev-only: MMA-thread wait cycles per CTA pair
    a.trace = reinterpret_cast<unsigned long long*>(strtoull(tr, nullptr, 0));
  if (const char* tr = getenv("MLRA_TRACE2"))  // dev-only: per-CTA timeline (globaltimer)
    a.trace2 = reinterpret_cast<unsigned long long*>(strtoull(tr, nullptr, 0));
  if (pair) {
    mlra::qgemm2_plan(a);
    if (a.sk_pairs) {  // stream-K: fp32 partial slots + zeroed publish flags
      a.sk_ws = sc.get<float>(static_cast<size_t>(a.sk_pairs * mlra::kSkSlotFloats));
      a.sk_flags = gp.sk_flags_zeroed ? gp.sk_flags_zeroed
                                      : sc.get<unsigned>(static_cast<size_t>(2 * a.sk_pairs));
      if (!a.sk_ws || !a.sk_flags) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
      if (!gp.sk_flags_zeroed)
        CUDA_TRY(cudaMemsetAsync(a.sk_flags, 0, 2 * a.sk_pairs * sizeof(unsigned), sc.st));
    }
    CUDA_TRY(mlra::qgemm2_launch(maps, d, a, w_tma, gp.mn, gp.out_f32, sc.st));
  }
  else
    CUDA_TRY(mlra::qgemm_launch(maps, d, a, w_tma, gp.mn, gp.out_f32, sc.st));
  return MLRA_OK;
}

// Workspace budget of one hook slab (bytes of bf16 Ŵ); MLRA_SLAB_MB overrides.
int64_t slab_budget() {
  int64_t mb = 256;
  if (const char* e = getenv("MLRA_SLAB_MB")) mb = atoll(e) > 0 ? atoll(e) : mb;
  return mb << 20;
}

// Slab extent along one side of Ŵ: a multiple of 256 (one pair tile), at least
// 256, covering `full` when `whole` (WeightMaterialize) or the budget allows.
int64_t slab_extent(int64_t full_pad, int64_t other_pad, bool whole) {
  if (whole) return full_pad;
  int64_t e = slab_budget() / (2 * other_pad) / 256 * 256;
  if (e < 256) e = 256;
  return e < full_pad ? e : full_pad;
}

// One bf16 tile through a plugin hook; a failing hook's status is returned
// with its name prepended to whatever message it left.
mlra_status call_hook(const mlra_hook* hk, const mlra_qweight* q, int64_t row0, int64_t nrows,
                      int64_t col0, int64_t ncols, void* out, int64_t ld, cudaStream_t st) {
  g_last_error.clear();
  const mlra_status rc = hk->materialize(hk->state, q, row0, nrows, col0, ncols, out, MLRA_BF16,
                                         ld, st);
  if (rc == MLRA_OK) return MLRA_OK;
  const std::string prev = g_last_error;
  return fail(rc, "quantizer hook '%s' failed (status %d)%s%s", hk->name ? hk->name : "?",
              static_cast<int>(rc), prev.empty() ? "" : ": ", prev.c_str());
}

// The hook path (the device Quantizer::matvec, lowprec_linear.cpp:174-182 /
// 226-235): Ŵ materialized through hk in slabs — rows for the forward (each
// slab's GEMM writes its own output columns), columns for dX (each slab's GEMM
// writes its own dX columns) — so no slab needs a cross-slab reduction.
mlra_status run_gemm_hooked(const mlra_qweight* q, const mlra_hook* hk, bool whole,
                            const GemmPlan& gp0, Scratch& sc) {
  const QWeightDev& d = q->d;
  if (!hk->materialize) return fail(MLRA_ERR_CONTRACT, "quantizer hook without materialize()");
  GemmPlan gp = gp0;
  gp.sk_flags_zeroed = nullptr;  // one zeroed flag set cannot serve several slab GEMMs
  const int64_t esize = gp.out_f32 ? 4 : 2;
  if (!gp.mn) {
    const int64_t slab = slab_extent(d.rows_pad, d.cols_pad, whole);
    auto* ws = sc.get<__nv_bfloat16>(static_cast<size_t>(slab * d.cols_pad));
    if (!ws) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
    for (int64_t r0 = 0; r0 < d.rows; r0 += slab) {
      const int64_t nr = d.rows - r0 < slab ? d.rows - r0 : slab;
      if (mlra_status st = call_hook(hk, q, r0, nr, 0, d.cols, ws, d.cols_pad, sc.st)) return st;
      QWeightDev v = d;
      v.rows = nr;
      v.rows_pad = round_up(nr, 256);
      GemmPlan g2 = gp;
      g2.out = static_cast<char*>(gp.out) + r0 * esize;
      if (gp.bias) g2.bias = gp.bias + r0;
      if (gp.w_lora) g2.w_lora = gp.w_lora + r0 * gp.rp;
      if (mlra_status st = run_gemm_d(v, ws, d.cols_pad, g2, sc)) return st;
    }
  } else {
    const int64_t slab = slab_extent(d.cols_pad, d.rows_pad, whole);
    auto* ws = sc.get<__nv_bfloat16>(static_cast<size_t>(d.rows * slab));
    if (!ws) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
    for (int64_t c0 = 0; c0 < d.cols; c0 += slab) {
      const int64_t nc = d.cols - c0 < slab ? d.cols - c0 : slab;
      if (mlra_status st = call_hook(hk, q, 0, d.rows, c0, nc, ws, slab, sc.st)) return st;
      QWeightDev v = d;
      v.cols = nc;
      v.cols_pad = round_up(nc, 256);
      GemmPlan g2 = gp;
      g2.out = static_cast<char*>(gp.out) + c0 * esize;
      if (gp.w_lora) g2.w_lora = gp.w_lora + c0 * gp.rp;
      if (mlra_status st = run_gemm_d(v, ws, slab, g2, sc)) return st;
    }
  }
  return MLRA_OK;
}

// Strategy dispatch (lowprec_linear.cpp:158-187): the hook is consulted under
// QuantizerMatvec only; an opaque qweight has nothing but its own hook.
const mlra_hook* pick_hook(const mlra_qweight* q, mlra_strategy strategy,
                           const mlra_hook* ctx_hook) {
  if (strategy == MLRA_MATVEC && ctx_hook) return ctx_hook;
  return q->opaque ? &q->hook : nullptr;
}

mlra_status run_gemm(const mlra_qweight* q, mlra_strategy strategy, const mlra_hook* ctx_hook,
                     const GemmPlan& gp, Scratch& sc) {
  // the built-in cb2 plugin decodes inside the fused GEMM (Ŵ never in HBM) for
  // the tile-materializing strategies unless a context hook overrides it
  if (q->opaque && q->cb2_fused && strategy != MLRA_WEIGHT &&
      !(strategy == MLRA_MATVEC && ctx_hook) && getenv("MLRA_CB2_HOOK") == nullptr) {
    GemmPlan g2 = gp;
    g2.cb2_codebook = q->cb2.codebook;
    g2.e8p = q->cb2.e8p;
    return run_gemm_d(q->cb2_d, nullptr, 0, g2, sc);
  }
  if (const mlra_hook* hk = pick_hook(q, strategy, ctx_hook))
    return run_gemm_hooked(q, hk, strategy == MLRA_WEIGHT, gp, sc);
  const QWeightDev& d = q->d;
  if (d.lut && strategy != MLRA_WEIGHT && mlra::qgemm_q_tma_ok(d)) {
    // the built-in lut plugin decodes inside the fused GEMM on the Q ring
    GemmPlan g2 = gp;
    g2.lut = d.lut;
    return run_gemm_d(d, nullptr, 0, g2, sc);
  }
  if (strategy == MLRA_WEIGHT || d.lut) {  // (lut groups the Q ring cannot tile: via HBM)
    // WeightMaterialize: the whole Ŵ in HBM for this pass (bf16), freed on return
    auto* w = sc.get<__nv_bfloat16>(static_cast<size_t>(d.rows * d.cols_pad));
    if (!w) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
    CUDA_TRY(mlra::launch_materialize(d, 0, d.rows, w, d.cols_pad, false, sc.st));
    return run_gemm_d(d, w, d.cols_pad, gp, sc);
  }
  return run_gemm_d(d, nullptr, 0, gp, sc);
}

mlra_status check_lora(const mlra_lora* L) {
  if (!L) return fail(MLRA_ERR_CONTRACT, "null layer");
  if (mlra_status st = check_q(L->q)) return st;
  if (L->rank < 1) return fail(MLRA_ERR_CONFIG, "adapter rank must be >= 1");
  if (!(L->alpha > 0.0)) return fail(MLRA_ERR_CONFIG, "adapter alpha must be positive");
  if (L->rank > 256) return fail(MLRA_ERR_CONFIG, "adapter rank %lld > 256 unsupported",
                                 (long long)L->rank);
  if (!L->a || !L->b) return fail(MLRA_ERR_CONTRACT, "adapter factors A/B missing");
  if (L->strategy < MLRA_WEIGHT || L->strategy > MLRA_MATVEC)
    return fail(MLRA_ERR_CONFIG, "unknown materialization strategy %d", (int)L->strategy);
  return MLRA_OK;
}

// Transposed hi/lo bf16 planes of an fp32 factor F [rows x r], one plane pair
// per 64-column chunk (thin_mma.cu consumes <= 64 columns per launch). The
// split jobs are queued on a PrepBatch, so they cost no launch of their own.
struct Planes {
  int n = 0;
  __nv_bfloat16* hi[4];
  __nv_bfloat16* lo[4];
  int64_t rc[4];
  int64_t rows_t[4];
  int64_t ldt = 0;
};

mlra_status alloc_planes(Scratch& sc, int64_t rows, int64_t r, bool ones, Planes* pl) {
  pl->ldt = round_up(rows, 64);
  pl->n = static_cast<int>((r + 63) / 64);
  for (int c = 0; c < pl->n; ++c) {
    const int64_t j0 = 64 * c, rc = r - j0 < 64 ? r - j0 : 64;
    const int64_t rows_t = mlra::thin_rows(rc, ones && c == 0);
    auto* hi = sc.get<__nv_bfloat16>(static_cast<size_t>(2 * rows_t * pl->ldt));
    if (!hi) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
    pl->hi[c] = hi;
    pl->lo[c] = hi + rows_t * pl->ldt;
    pl->rc[c] = rc;
    pl->rows_t[c] = rows_t;
  }
  return MLRA_OK;
}

mlra_status make_planes(Scratch& sc, mlra::PrepBatch& pb, const float* F, int64_t rows, int64_t r,
                        bool ones, Planes* pl) {
  if (mlra_status st = alloc_planes(sc, rows, r, ones, pl)) return st;
  for (int c = 0; c < pl->n; ++c)
    pb.split_t(F + 64 * c, rows, pl->rc[c], r, ones && c == 0, pl->hi[c], pl->lo[c],
               pl->rows_t[c], pl->ldt);
  return MLRA_OK;
}

// Workspace of a skinny product (partial slots + per-tile counters); the
// counters are zeroed by the pass's prep launch and reset by the finishers, so
// every chunk launch of the pass (same stream) reuses them.
struct ThinWs {
  float* ws = nullptr;
  int64_t ws_floats = 0;
  int* cnt = nullptr;
};
mlra_status thin_ws(Scratch& sc, mlra::PrepBatch& pb, bool row, int64_t m, int64_t d, int64_t r,
                    bool ones, ThinWs* w) {
  int64_t wf = 0, nc = 0;
  for (int64_t j0 = 0; j0 < r; j0 += 64) {  // the largest chunk's needs
    int64_t f, c;
    mlra::thin_ws_size(row, m, d, r - j0 < 64 ? r - j0 : 64, ones && j0 == 0, &f, &c);
    wf = f > wf ? f : wf;
    nc = c > nc ? c : nc;
  }
  w->ws = sc.get<float>(static_cast<size_t>(wf));
  w->ws_floats = wf;
  w->cnt = sc.get<int>(static_cast<size_t>(nc));
  if (!w->ws || !w->cnt) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  pb.zero_f32(reinterpret_cast<float*>(w->cnt), nc);
  return MLRA_OK;
}

// Publish flags for a stream-K / split-K GEMM of this pass (the most any plan
// uses), zeroed by the pass's prep launch.
unsigned* gemm_flags(Scratch& sc, mlra::PrepBatch& pb) {
  constexpr int64_t n = 2 * mlra::kMaxSkPairs;
  auto* f = sc.get<unsigned>(static_cast<size_t>(n));
  if (f) pb.zero_f32(reinterpret_cast<float*>(f), n);
  return f;
}

// dev-only per-CTA timeline of the skinny kernels (MLRA_TRACE3 = device pointer
// to 8 x CTAs u64, used only by a -DMLRA_DEV_TRACE build)
unsigned long long* thin_trace() {
  const char* e = getenv("MLRA_TRACE3");
  return e ? reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 0)) : nullptr;
}

// out[m x r] = act[m x kd] · W   (K4 / K5a; W as planes). Optionally also the
// padded bf16(pad_scale · out) operand [m x rp] and the transposed hi/lo planes
// of out (tp, allocated by alloc_planes over m rows).
mlra_status rows_product(cudaStream_t st, const ThinWs& w, const __nv_bfloat16* act, int64_t lda,
                         int64_t m, int64_t kd, const Planes& W, float* out, int64_t r,
                         __nv_bfloat16* pad, int64_t rp, float pad_scale, const Planes* tp) {
  for (int c = 0; c < W.n; ++c) {
    mlra::ThinOut o;
    o.out = out + 64 * c;
    o.ldo = r;
    o.ws = w.ws;
    o.ws_floats = w.ws_floats;
    o.cnt = w.cnt;
    if (pad) {
      o.pad = pad + 64 * c;
      o.ldp = rp;
      o.pad_cols = 64;
      o.pad_scale = pad_scale;
    }
    o.trace = thin_trace();
    if (tp) {
      o.thi = tp->hi[c];
      o.ldt = tp->ldt;
      o.t_rows = static_cast<int>(tp->rows_t[c]);
    }
    CUDA_TRY(mlra::launch_rowmma(act, lda, m, kd, W.hi[c], W.lo[c], W.ldt, W.rc[c], o, st));
  }
  return MLRA_OK;
}

// out[nd x r] = scale · actᵀ · V  (+ colsum[n] = Σ_t act[t, n])  (K5b / K6)
mlra_status cols_product(cudaStream_t st, const ThinWs& w, const __nv_bfloat16* act, int64_t lda,
                         int64_t m, int64_t nd, const Planes& V, float scale, float* out,
                         int64_t r, float* colsum) {
  for (int c = 0; c < V.n; ++c) {
    mlra::ThinOut o;
    o.out = out + 64 * c;
    o.ldo = r;
    o.scale = scale;
    o.colsum = c == 0 ? colsum : nullptr;
    o.trace = thin_trace();
    o.ws = w.ws;
    o.ws_floats = w.ws_floats;
    o.cnt = w.cnt;
    CUDA_TRY(mlra::launch_colmma(act, lda, m, nd, V.hi[c], V.lo[c], V.ldt, V.rc[c], o, st));
  }
  return MLRA_OK;
}

// Per-thread, per-device side stream: the dA/dB products of a backward pass run
// on it concurrently with the dX GEMM (they fill the SMs its last tile wave
// leaves idle) and are joined back to the caller's stream before return.
struct SideStream {
  cudaStream_t st = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, mid = nullptr;
};
mlra_status side_stream(SideStream** out) {
  thread_local SideStream per_dev[64];
  int dev = 0;
  CUDA_TRY(cudaGetDevice(&dev));
  if (dev >= 64) return fail(MLRA_ERR_UNSUPPORTED, "device index %d", dev);
  SideStream& ss = per_dev[dev];
  if (!ss.st) {
    CUDA_TRY(cudaStreamCreateWithFlags(&ss.st, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(&ss.mid, cudaEventDisableTiming));
  }
  *out = &ss;
  return MLRA_OK;
}


// The E8P abs-pattern table (QuIP#'s E8P12 construction): (i) every vector in
// {1/2, 3/2, 5/2}^8 with squared norm <= 10, in lexicographic order of 2|a|
// (227 patterns), then (ii) 29 patterns of squared norm 12 with entries in
// {1/2, 3/2}; odd bit i = the coordinate sum of pattern i is odd. Restated in
// oracle/mlra_oracle.c (orc_e8p_abs_table).
void e8p_abs_table(float (*a)[8], uint32_t* odd) {
  static const uint8_t kNorm12[29][8] = {
      {3, 1, 1, 1, 3, 3, 3, 3}, {1, 3, 1, 1, 3, 3, 3, 3}, {1, 1, 3, 1, 3, 3, 3, 3},
      {1, 1, 1, 3, 3, 3, 3, 3}, {3, 3, 3, 1, 3, 3, 1, 1}, {3, 3, 3, 1, 3, 1, 3, 1},
      {3, 3, 3, 1, 1, 3, 3, 1}, {3, 3, 3, 1, 3, 1, 1, 3}, {3, 3, 3, 1, 1, 3, 1, 3},
      {3, 3, 3, 1, 1, 1, 3, 3}, {3, 3, 1, 3, 3, 3, 1, 1}, {3, 3, 1, 3, 3, 1, 3, 1},
      {3, 3, 1, 3, 1, 3, 3, 1}, {3, 3, 1, 3, 3, 1, 1, 3}, {3, 3, 1, 3, 1, 3, 1, 3},
      {3, 3, 1, 3, 1, 1, 3, 3}, {3, 1, 3, 3, 3, 3, 1, 1}, {3, 1, 3, 3, 3, 1, 3, 1},
      {3, 1, 3, 3, 1, 3, 3, 1}, {3, 1, 3, 3, 3, 1, 1, 3}, {3, 1, 3, 3, 1, 3, 1, 3},
      {1, 3, 3, 3, 1, 1, 3, 3}, {1, 3, 3, 3, 3, 3, 1, 1}, {1, 3, 3, 3, 3, 1, 3, 1},
      {1, 3, 3, 3, 1, 3, 3, 1}, {1, 3, 3, 3, 3, 1, 1, 3}, {1, 3, 3, 3, 1, 3, 1, 3},
      {1, 1, 3, 3, 1, 3, 3, 3}, {3, 3, 1, 1, 3, 3, 3, 1}};
  int n = 0;
  for (int c = 0; c < 6561 && n < 227; ++c) {  // base-3 digits, most significant first
    int d[8], v = c, norm4 = 0;
    for (int j = 7; j >= 0; --j) {
      d[j] = 2 * (v % 3) + 1;  // 1, 3, 5 = 2|a|
      v /= 3;
      norm4 += d[j] * d[j];
    }
    if (norm4 > 40) continue;
    for (int j = 0; j < 8; ++j) a[n][j] = 0.5f * static_cast<float>(d[j]);
    ++n;
  }
  for (int i = 0; i < 29; ++i, ++n)
    for (int j = 0; j < 8; ++j) a[n][j] = 0.5f * static_cast<float>(kNorm12[i][j]);
  for (int w = 0; w < 8; ++w) odd[w] = 0u;
  for (int i = 0; i < 256; ++i) {
    int twice = 0;  // 2 * coordinate sum
    for (int j = 0; j < 8; ++j) twice += static_cast<int>(2.0f * a[i][j]);
    if ((twice / 2) & 1) odd[i >> 5] |= 1u << (i & 31);
  }
}

// Shared by the codebook plugins (cb2, e8p): validation, an opaque qweight whose
// hook is k_cb2_materialize, the device codebook/codes/scales upload and, for
// whole 256-multiples, the fused Q-ring view of the u16 code stream.
mlra_status codebook_qweight_create(const char* name, int64_t rows, int64_t cols, int64_t group,
                                    const uint16_t* codes, const std::vector<uint32_t>& cbdev,
                                    bool cb16, bool e8p, const float* scales, void* stream,
                                    mlra_qweight** out) {
  if (!out) return fail(MLRA_ERR_CONTRACT, "null output handle");
  *out = nullptr;
  if (rows <= 0 || cols <= 0 || cols % 8 != 0)
    return fail(MLRA_ERR_CONFIG, "%s: cols %lld must be a positive multiple of 8", name,
                (long long)cols);
  if (group <= 0 || group % 8 != 0 || cols % group != 0)
    return fail(MLRA_ERR_CONFIG, "%s: group size %lld must be a multiple of 8 dividing cols %lld",
                name, (long long)group, (long long)cols);
  if (!codes || !scales) return fail(MLRA_ERR_CONTRACT, "%s: null buffers", name);
  const int64_t ng = rows * (cols / group);
  for (int64_t i = 0; i < ng; ++i)
    if (!(scales[i] > 0.0f)) return fail(MLRA_ERR_NUMERIC, "%s: non-positive scale", name);
  if (mlra_status st = check_device()) return st;
  static const auto kHookFn = [](void*, const mlra_qweight* q, int64_t row0, int64_t nrows,
                                 int64_t col0, int64_t ncols, void* o, mlra_dtype dtype,
                                 int64_t ld, void* st) -> mlra_status {
    if (col0 % 8 != 0 || ncols % 8 != 0)
      return fail(MLRA_ERR_RANGE, "%s: tile columns must be 8-aligned", q->hook_name.c_str());
    CUDA_TRY(mlra::launch_cb2_materialize(q->cb2, row0, nrows, col0, ncols, o, ld,
                                          dtype == MLRA_F32, static_cast<cudaStream_t>(st)));
    return MLRA_OK;
  };
  static const mlra_hook kCb2Hook = {"cb2", nullptr, kHookFn};
  static const mlra_hook kE8pHook = {"e8p", nullptr, kHookFn};
  mlra_qweight* q = nullptr;
  if (mlra_status st = mlra_qweight_create_opaque(rows, cols, 2, e8p ? &kE8pHook : &kCb2Hook, &q))
    return st;
  const size_t cb_bytes = cbdev.size() * 4, code_bytes = static_cast<size_t>(rows * (cols / 8)) * 2,
               sc_bytes = static_cast<size_t>(ng) * 4;
  const size_t off_codes = cb_bytes, off_sc = round_up(off_codes + code_bytes, 16);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMalloc(&q->cb2_mem, off_sc + sc_bytes);
  char* base = static_cast<char*>(q->cb2_mem);
  if (e == cudaSuccess) e = cudaMemcpyAsync(base, cbdev.data(), cb_bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(base + off_codes, codes, code_bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(base + off_sc, scales, sc_bytes, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    mlra_qweight_destroy(q);
    return fail(MLRA_ERR_CUDA, "%s upload: %s", name, cudaGetErrorString(e));
  }
  q->device_bytes = off_sc + sc_bytes;
  q->d.group = group;
  // fused path: whole 256-multiples (the u16 codes are then the row-aligned 2-bit
  // stream the Q ring tiles), a bf16-exact codebook, a group the Q ring supports
  const bool g_ok = group == 32 || group == 64 || group % 128 == 0;
  if (cb16 && g_ok && rows % 256 == 0 && cols % 256 == 0) {
    QWeightDev& fd = q->cb2_d;
    fd.rows = fd.rows_pad = rows;
    fd.cols = fd.cols_pad = cols;
    fd.bits = 2;
    fd.group = group;
    fd.ng_pad = round_up(cols / group, 2);
    fd.row_words = cols / 16;
    fd.words = reinterpret_cast<const uint32_t*>(base + off_codes);
    std::vector<float2> g(static_cast<size_t>(rows * fd.ng_pad), make_float2(1.0f, 0.0f));
    for (int64_t i = 0; i < rows; ++i)
      for (int64_t j = 0; j < cols / group; ++j)
        g[static_cast<size_t>(i * fd.ng_pad + j)] = make_float2(scales[i * (cols / group) + j], 0.0f);
    e = cudaMalloc(&q->cb2_grid, g.size() * sizeof(float2));
    if (e == cudaSuccess)
      e = cudaMemcpy(q->cb2_grid, g.data(), g.size() * sizeof(float2), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      mlra_qweight_destroy(q);
      return fail(MLRA_ERR_CUDA, "%s grid upload: %s", name, cudaGetErrorString(e));
    }
    fd.grid = q->cb2_grid;
    q->device_bytes += g.size() * sizeof(float2);
    q->cb2_fused = true;
  }
  q->cb2 = mlra::Cb2Dev{rows, cols, group, cols / group,
                        reinterpret_cast<const uint16_t*>(base + off_codes), base, cb16 ? 1 : 0,
                        reinterpret_cast<const float*>(base + off_sc), e8p ? 1 : 0};
  *out = q;
  return MLRA_OK;
}
}  // namespace

extern "C" {

const char* mlra_last_error(void) { return g_last_error.c_str(); }
int mlra_last_format_error(uint64_t* offset) {
  if (offset) *offset = g_format_offset;
  return g_format_kind;
}
int mlra_abi_version(void) { return 2; }
uint64_t mlra_kernel_launches(void) { return mlra::g_launches.load(); }
mlra_status mlra_device_check(void) { return check_device(); }

uint64_t mlra_packed_word_count(uint64_t count, int bits) {
  return (count * static_cast<uint64_t>(bits) + 31) / 32;
}

mlra_status mlra_qweight_create(int64_t rows, int64_t cols, int bits, int64_t group,
                                const uint32_t* words, uint64_t word_count,
                                uint64_t code_count, const float* scales, const float* zeros,
                                uint64_t grid_count, void* stream, mlra_qweight** out) {
  if (!out) return fail(MLRA_ERR_CONTRACT, "null output handle");
  *out = nullptr;
  // QuantizedMatrix::validate — quantize.cpp:82-115 (same order, same types)
  if (!supported_bits(bits))
    return fail(MLRA_ERR_CONFIG, "QuantizedMatrix: unsupported bit width %d", bits);
  if (rows <= 0 || cols <= 0 || group <= 0 || cols % group != 0)
    return fail(MLRA_ERR_CONFIG, "QuantizedMatrix: group size %lld does not divide cols %lld",
                (long long)group, (long long)cols);
  if (code_count != static_cast<uint64_t>(rows * cols))
    return fail(MLRA_ERR_FORMAT, "QuantizedMatrix: code count %llu != rows*cols",
                (unsigned long long)code_count);
  const uint64_t ng = static_cast<uint64_t>(rows * (cols / group));
  if (grid_count != ng)
    return fail(MLRA_ERR_FORMAT, "QuantizedMatrix: grid count mismatch (%llu, expected %llu)",
                (unsigned long long)grid_count, (unsigned long long)ng);
  if (!words || !scales || !zeros) return fail(MLRA_ERR_CONTRACT, "null weight buffers");
  for (uint64_t i = 0; i < ng; ++i)
    if (!(scales[i] > 0.0f)) return fail(MLRA_ERR_NUMERIC, "QuantizedMatrix: non-positive scale");
  // bitpack validate_metadata — bitpack.cpp:37-60
  const uint64_t expect = mlra_packed_word_count(code_count, bits);
  if (word_count != expect)
    return fail(MLRA_ERR_FORMAT,
                "bitpack: corrupted length metadata: %llu words for %llu codes at %d bits "
                "(expected %llu)",
                (unsigned long long)word_count, (unsigned long long)code_count, bits,
                (unsigned long long)expect);
  const uint64_t tail = word_count * 32 - code_count * bits;
  if (word_count && tail > 0 && tail < 32 && (words[word_count - 1] >> (32 - tail)) != 0)
    return fail(MLRA_ERR_FORMAT, "bitpack: nonzero trailing bits in last word");
  if (mlra_status st = check_device()) return st;

  cudaStream_t s = static_cast<cudaStream_t>(stream);
  auto* q = new mlra_qweight();
  QWeightDev& d = q->d;
  d.rows = rows;
  d.cols = cols;
  d.rows_pad = round_up(rows, 256);
  d.cols_pad = round_up(cols, 256);
  d.bits = bits;
  d.group = group;
  d.ng_pad = round_up((d.cols_pad + group - 1) / group, 2);  // even: 16-B grid rows for TMA
  d.row_words = d.cols_pad * bits / 32;
  const size_t nwords = static_cast<size_t>(d.rows_pad * d.row_words) + 4;
  const size_t ngrid = static_cast<size_t>(d.rows_pad * d.ng_pad);
  auto cleanup = [&](mlra_status st) {
    if (q->words) cudaFree(q->words);
    if (q->grid) cudaFree(q->grid);
    delete q;
    return st;
  };
  if (cudaMalloc(&q->words, nwords * 4) != cudaSuccess ||
      cudaMalloc(&q->grid, ngrid * sizeof(float2)) != cudaSuccess)
    return cleanup(fail(MLRA_ERR_CUDA, "device allocation of %zu bytes failed",
                        nwords * 4 + ngrid * 8));
  q->device_bytes = nwords * 4 + ngrid * sizeof(float2);
  d.words = q->words;
  d.grid = q->grid;

  uint32_t* src_words = nullptr;
  float *dsc = nullptr, *dz = nullptr;
  int* dcount = nullptr;
  auto tmpfree = [&]() {
    if (src_words) cudaFree(src_words);
    if (dsc) cudaFree(dsc);
    if (dz) cudaFree(dz);
    if (dcount) cudaFree(dcount);
  };
  cudaError_t e = cudaSuccess;
  const bool verbatim = (d.rows_pad == rows) && (d.cols_pad == cols);
  if (verbatim) {
    e = cudaMemcpyAsync(q->words, words, word_count * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(q->words + word_count, 0, 16, s);
  } else {
    e = cudaMalloc(&src_words, (word_count + 2) * 4);
    if (e == cudaSuccess) e = cudaMemsetAsync(src_words, 0, (word_count + 2) * 4, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(src_words, words, word_count * 4, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess)
      e = mlra::launch_relayout(src_words, rows, cols, bits, d.row_words, d.rows_pad, q->words, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(q->words + d.rows_pad * d.row_words, 0, 16, s);
  }
  if (e == cudaSuccess) e = cudaMalloc(&dsc, ng * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dz, ng * 4);
  if (e == cudaSuccess) e = cudaMalloc(&dcount, sizeof(int));
  if (e == cudaSuccess) e = cudaMemcpyAsync(dsc, scales, ng * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dz, zeros, ng * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(dcount, 0, sizeof(int), s);
  if (e == cudaSuccess)
    e = mlra::launch_grid(dsc, dz, rows, cols / group, d.rows_pad, d.ng_pad, bits, q->grid,
                          dcount, s);
  int unc = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&unc, dcount, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  tmpfree();
  if (e != cudaSuccess)
    return cleanup(fail(MLRA_ERR_CUDA, "qweight upload: %s", cudaGetErrorString(e)));
  q->uncertified = unc;
  *out = q;
  return MLRA_OK;
}

void mlra_qweight_destroy(mlra_qweight* q) {
  if (!q) return;
  if (q->words) cudaFree(q->words);
  if (q->grid) cudaFree(q->grid);
  if (q->cb2_mem) cudaFree(q->cb2_mem);
  if (q->cb2_grid) cudaFree(q->cb2_grid);
  if (q->lut_mem) cudaFree(q->lut_mem);
  delete q;
}

mlra_status mlra_qweight_create_opaque(int64_t rows, int64_t cols, int bits,
                                       const mlra_hook* hook, mlra_qweight** out) {
  if (!out) return fail(MLRA_ERR_CONTRACT, "null output handle");
  *out = nullptr;
  if (!hook || !hook->materialize)
    return fail(MLRA_ERR_CONTRACT, "opaque qweight: hook with materialize() required");
  if (rows <= 0 || cols <= 0)
    return fail(MLRA_ERR_CONFIG, "QuantizedMatrix: empty shape %lld x %lld", (long long)rows,
                (long long)cols);
  if (bits < 1 || bits > 16) return fail(MLRA_ERR_CONFIG, "unsupported bit width %d", bits);
  auto* q = new mlra_qweight();
  q->opaque = true;
  q->hook = *hook;
  q->hook_name = hook->name ? hook->name : "";
  q->hook.name = q->hook_name.c_str();
  QWeightDev& d = q->d;
  d.rows = rows;
  d.cols = cols;
  d.rows_pad = round_up(rows, 256);
  d.cols_pad = round_up(cols, 256);
  d.bits = bits;
  d.group = cols;
  *out = q;
  return MLRA_OK;
}

mlra_status mlra_cb2_create(int64_t rows, int64_t cols, int64_t group, const uint16_t* codes,
                            const float* codebook, const float* scales, void* stream,
                            mlra_qweight** out) {
  if (!codebook) return fail(MLRA_ERR_CONTRACT, "cb2: null buffers");
  for (int i = 0; i < 256 * 8; ++i)
    if (!(codebook[i] >= 0.0f) || codebook[i] > 3.4e38f)
      return fail(MLRA_ERR_NUMERIC, "cb2: codebook magnitudes must be finite and >= 0");
  // device codebook layout (common.cuh Cb2Dev): bf16-exact magnitudes -> 8 bf16
  // per code, else the two float4 halves in separate arrays
  bool cb16 = true;
  for (int i = 0; i < 256 * 8 && cb16; ++i) {
    uint32_t u;
    std::memcpy(&u, &codebook[i], 4);
    cb16 = (u & 0xFFFFu) == 0;
  }
  std::vector<uint32_t> cbdev(cb16 ? 256 * 4 : 256 * 8);
  for (int i = 0; i < 256; ++i)
    for (int e = 0; e < 8; ++e) {
      uint32_t u;
      std::memcpy(&u, &codebook[i * 8 + e], 4);
      if (cb16)
        cbdev[i * 4 + e / 2] |= (u >> 16) << (16 * (e & 1));
      else
        cbdev[(e / 4) * 1024 + i * 4 + (e & 3)] = u;
    }
  return codebook_qweight_create("cb2", rows, cols, group, codes, cbdev, cb16, false, scales,
                                 stream, out);
}

int mlra_e8p_abs_table(float* abs_out, uint32_t* odd_out) {
  float a[256][8];
  uint32_t odd[8];
  e8p_abs_table(a, odd);
  if (abs_out) std::memcpy(abs_out, a, sizeof(a));
  if (odd_out) std::memcpy(odd_out, odd, sizeof(odd));
  return 256;
}

mlra_status mlra_e8p_create(int64_t rows, int64_t cols, int64_t group, const uint16_t* codes,
                            const float* scales, void* stream, mlra_qweight** out) {
  // device tables: bf16 rows of (|a| + 1/4), then of (|a| - 1/4), then the odd bits
  float a[256][8];
  uint32_t odd[8];
  e8p_abs_table(a, odd);
  std::vector<uint32_t> tab(2 * 256 * 4 + 32 / 4, 0u);
  for (int h = 0; h < 2; ++h)
    for (int i = 0; i < 256; ++i)
      for (int e = 0; e < 8; ++e) {
        const float m = a[i][e] + (h == 0 ? 0.25f : -0.25f);  // exact (multiples of 1/4)
        uint32_t u;
        std::memcpy(&u, &m, 4);
        tab[h * 1024 + i * 4 + e / 2] |= (u >> 16) << (16 * (e & 1));
      }
  for (int w = 0; w < 8; ++w) tab[2048 + w] = odd[w];
  return codebook_qweight_create("e8p", rows, cols, group, codes, tab, true, true, scales, stream,
                                 out);
}

mlra_status mlra_lut_create(int64_t rows, int64_t cols, int bits, int64_t group,
                            const uint32_t* words, uint64_t word_count, const float* levels,
                            const float* scales, void* stream, mlra_qweight** out) {
  if (!out) return fail(MLRA_ERR_CONTRACT, "null output handle");
  *out = nullptr;
  if (bits != 2 && bits != 3 && bits != 4)
    return fail(MLRA_ERR_CONFIG, "lut: unsupported bit width %d (2, 3 or 4)", bits);
  if (rows <= 0 || cols <= 0 || group <= 0 || group % 8 != 0 || cols % group != 0)
    return fail(MLRA_ERR_CONFIG, "lut: group size %lld must be a multiple of 8 dividing cols %lld",
                (long long)group, (long long)cols);
  if (!words || !levels || !scales) return fail(MLRA_ERR_CONTRACT, "lut: null buffers");
  const int nl = 1 << bits;
  for (int i = 0; i < nl; ++i)
    if (!std::isfinite(levels[i])) return fail(MLRA_ERR_NUMERIC, "lut: level %d is not finite", i);
  const uint64_t ng = static_cast<uint64_t>(rows * (cols / group));
  for (uint64_t i = 0; i < ng; ++i)
    if (!(scales[i] > 0.0f) || !std::isfinite(scales[i]))
      return fail(MLRA_ERR_NUMERIC, "lut: scales must be positive and finite");
  // the codes and scales go through the affine upload with zero = 0 (its grid
  // is then {s, 0}, every group certified: s·c is exact in f64); the table
  // replaces the affine decode
  std::vector<float> zeros(ng, 0.0f);
  mlra_qweight* q = nullptr;
  if (mlra_status st = mlra_qweight_create(rows, cols, bits, group, words, word_count,
                                           static_cast<uint64_t>(rows * cols), scales,
                                           zeros.data(), ng, stream, &q))
    return st;
  float table[16] = {};
  std::memcpy(table, levels, nl * sizeof(float));
  cudaError_t e = cudaMalloc(&q->lut_mem, sizeof(table));
  if (e == cudaSuccess) e = cudaMemcpy(q->lut_mem, table, sizeof(table), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    mlra_qweight_destroy(q);
    return fail(MLRA_ERR_CUDA, "lut upload: %s", cudaGetErrorString(e));
  }
  q->d.lut = q->lut_mem;
  q->device_bytes += sizeof(table);
  *out = q;
  return MLRA_OK;
}

mlra_status mlra_quantize_rtn(const void* w, mlra_dtype dtype, int64_t rows, int64_t cols,
                              int bits, int64_t group, uint32_t* words, float* scales,
                              float* zeros, void* stream) {
  // validate_quantize_args (quantize.cpp:46-59), group 0 = per row (:78-80)
  if (group == 0) group = cols;
  if (rows <= 0 || cols <= 0) return fail(MLRA_ERR_DIMENSION, "quantize: matrix must be non-empty");
  if (!supported_bits(bits))
    return fail(MLRA_ERR_CONFIG, "quantize: unsupported bit width %d", bits);
  if (group <= 0 || cols % group != 0)
    return fail(MLRA_ERR_CONFIG, "quantize: group size %lld does not divide cols %lld",
                (long long)group, (long long)cols);
  if (dtype != MLRA_F64 && dtype != MLRA_F32)
    return fail(MLRA_ERR_CONFIG, "quantize: weights must be f64 or f32");
  if (!w || !words || !scales || !zeros) return fail(MLRA_ERR_CONTRACT, "quantize: null buffers");
  if (mlra_status st = check_device()) return st;
  const uint64_t nwords = mlra_packed_word_count(static_cast<uint64_t>(rows * cols), bits);
  CUDA_TRY(mlra::launch_quantize_rtn(w, dtype == MLRA_F64, rows, cols, group, bits, words, nwords,
                                     scales, zeros, static_cast<cudaStream_t>(stream)));
  return MLRA_OK;
}

mlra_status mlra_optq_workspace(const double* calib, int64_t m, int64_t dim, double damping,
                                double* hessian, double* upper, void* stream) {
  // build_optq_workspace (quantize.cpp:186-211)
  if (m <= 0 || dim <= 0)
    return fail(MLRA_ERR_DIMENSION, "optq: calibration must be [m x %lld], got %lldx%lld",
                (long long)dim, (long long)m, (long long)dim);
  if (!(damping >= 0.0)) return fail(MLRA_ERR_CONFIG, "optq: damping must be non-negative");
  if (!calib || !hessian || !upper) return fail(MLRA_ERR_CONTRACT, "optq: null buffers");
  if (mlra_status st = check_device()) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* scratch = nullptr;
  int* bad = nullptr;
  CUDA_TRY(cudaMallocAsync(&scratch, 2 * dim * dim * sizeof(double), s));
  cudaError_t e = cudaMallocAsync(&bad, 2 * sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(bad, 0x7f, 2 * sizeof(int), s);
  if (e == cudaSuccess)
    e = mlra::launch_optq_workspace(calib, m, dim, damping, hessian, upper, scratch, bad, s);
  int hb[2] = {0x7f7f7f7f, 0x7f7f7f7f};
  if (e == cudaSuccess) e = cudaMemcpyAsync(hb, bad, sizeof(hb), cudaMemcpyDeviceToHost, s);
  cudaFreeAsync(scratch, s);
  if (bad) cudaFreeAsync(bad, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(MLRA_ERR_CUDA, "optq workspace: %s", cudaGetErrorString(e));
  if (hb[0] < dim || hb[1] < dim)
    return fail(MLRA_ERR_NUMERIC, "optq: calibration Hessian not invertible after damping");
  return MLRA_OK;
}

mlra_status mlra_quantize_optq(const double* w, const double* calib, int64_t rows, int64_t cols,
                               int64_t m, int bits, int64_t group, double damping, uint32_t* words,
                               float* scales, float* zeros, void* stream) {
  // quantize_optq (quantize.cpp:213-255): normalize_group_size, validate_quantize_args,
  // build_optq_workspace, grids from the original weights, the column sweep
  if (group == 0) group = cols;
  if (rows <= 0 || cols <= 0) return fail(MLRA_ERR_DIMENSION, "quantize: matrix must be non-empty");
  if (!supported_bits(bits))
    return fail(MLRA_ERR_CONFIG, "quantize: unsupported bit width %d", bits);
  if (group <= 0 || cols % group != 0)
    return fail(MLRA_ERR_CONFIG, "quantize: group size %lld does not divide cols %lld",
                (long long)group, (long long)cols);
  if (!w || !words || !scales || !zeros) return fail(MLRA_ERR_CONTRACT, "optq: null buffers");
  if (mlra_status st = check_device()) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double *h = nullptr, *u = nullptr, *es = nullptr;
  uint32_t* codes = nullptr;
  auto release = [&]() {
    if (h) cudaFreeAsync(h, s);
    if (u) cudaFreeAsync(u, s);
    if (es) cudaFreeAsync(es, s);
    if (codes) cudaFreeAsync(codes, s);
  };
  if (cudaMallocAsync(&h, cols * cols * sizeof(double), s) != cudaSuccess ||
      cudaMallocAsync(&u, cols * cols * sizeof(double), s) != cudaSuccess) {
    release();
    return fail(MLRA_ERR_CUDA, "optq: workspace allocation failed");
  }
  if (mlra_status st = mlra_optq_workspace(calib, m, cols, damping, h, u, stream)) {
    release();
    return st;
  }
  const uint64_t nwords = mlra_packed_word_count(static_cast<uint64_t>(rows * cols), bits);
  cudaError_t e = cudaMallocAsync(&es, rows * cols * sizeof(double), s);
  if (e == cudaSuccess) e = cudaMallocAsync(&codes, rows * cols * sizeof(uint32_t), s);
  if (e == cudaSuccess) e = mlra::launch_rtn_grid(w, rows, cols, group, bits, scales, zeros, s);
  if (e == cudaSuccess)
    e = mlra::launch_optq_sweep(w, u, rows, cols, group, bits, scales, zeros, es, codes, words,
                                nwords, s);
  release();
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(MLRA_ERR_CUDA, "optq: %s", cudaGetErrorString(e));
  return MLRA_OK;
}

const mlra_hook* mlra_qweight_hook(const mlra_qweight* q) {
  return q && q->opaque ? &q->hook : nullptr;
}

mlra_status mlra_qweight_info(const mlra_qweight* q, int64_t* rows, int64_t* cols, int* bits,
                              int64_t* group, uint64_t* device_bytes, int64_t* uncertified) {
  if (mlra_status st = check_q(q)) return st;
  if (rows) *rows = q->d.rows;
  if (cols) *cols = q->d.cols;
  if (bits) *bits = q->d.bits;
  if (group) *group = q->d.group;
  if (device_bytes) *device_bytes = q->device_bytes;
  if (uncertified) *uncertified = q->uncertified;
  return MLRA_OK;
}

uint64_t mlra_ledger_bytes(const mlra_qweight* q, mlra_strategy strategy) {
  if (!q) return 0;
  if (strategy == MLRA_WEIGHT)
    return static_cast<uint64_t>(q->d.rows) * static_cast<uint64_t>(q->d.cols) * 2u;
  if (q->d.lut && !mlra::qgemm_q_tma_ok(q->d))  // lut groups off the Q ring: whole Ŵ
    return static_cast<uint64_t>(q->d.rows) * static_cast<uint64_t>(q->d.cols) * 2u;
  if (!q->opaque || q->cb2_fused) return 0;
  // hook slabs: the larger of the forward (row) and dX (column) slab buffers
  const QWeightDev& d = q->d;
  const int64_t fwd = slab_extent(d.rows_pad, d.cols_pad, false) * d.cols_pad;
  const int64_t bwd = slab_extent(d.cols_pad, d.rows_pad, false) * d.rows;
  return static_cast<uint64_t>(fwd > bwd ? fwd : bwd) * 2u;
}

mlra_status mlra_materialize_rows(const mlra_qweight* q, int64_t row0, int64_t nrows, void* out,
                                  mlra_dtype dtype, int64_t ld, void* stream) {
  if (mlra_status st = check_q(q)) return st;
  if (row0 < 0 || nrows < 0 || row0 + nrows > q->d.rows)
    return fail(MLRA_ERR_RANGE, "dequantize_row: rows [%lld, %lld) out of range [0, %lld)",
                (long long)row0, (long long)(row0 + nrows), (long long)q->d.rows);
  if (ld < q->d.cols)
    return fail(MLRA_ERR_DIMENSION, "dequantize_into: buffer size mismatch (ld %lld < cols %lld)",
                (long long)ld, (long long)q->d.cols);
  return mlra_materialize_tile(q, row0, nrows, 0, q->d.cols, out, dtype, ld, stream);
}

mlra_status mlra_materialize_tile(const mlra_qweight* q, int64_t row0, int64_t nrows,
                                  int64_t col0, int64_t ncols, void* out, mlra_dtype dtype,
                                  int64_t ld, void* stream) {
  if (mlra_status st = check_q(q)) return st;
  if (row0 < 0 || nrows < 0 || row0 + nrows > q->d.rows)
    return fail(MLRA_ERR_RANGE, "dequantize_row: rows [%lld, %lld) out of range [0, %lld)",
                (long long)row0, (long long)(row0 + nrows), (long long)q->d.rows);
  if (col0 < 0 || ncols < 0 || col0 + ncols > q->d.cols || col0 % 8 != 0)
    return fail(MLRA_ERR_RANGE, "materialize_tile: cols [%lld, %lld) out of range [0, %lld) "
                "or not 8-aligned", (long long)col0, (long long)(col0 + ncols),
                (long long)q->d.cols);
  if (ld < ncols)
    return fail(MLRA_ERR_DIMENSION, "dequantize_into: buffer size mismatch (ld %lld < cols %lld)",
                (long long)ld, (long long)ncols);
  if (dtype != MLRA_F32 && dtype != MLRA_BF16) return fail(MLRA_ERR_CONFIG, "bad dtype");
  if (mlra_status st = check_device()) return st;
  if (nrows == 0 || ncols == 0) return MLRA_OK;
  if (q->opaque) {
    if (!q->hook.materialize) return fail(MLRA_ERR_CONTRACT, "opaque qweight without a hook");
    return q->hook.materialize(q->hook.state, q, row0, nrows, col0, ncols, out, dtype, ld,
                               stream);
  }
  if (q->d.lut && ncols % 8 != 0)
    return fail(MLRA_ERR_RANGE, "lut: tile columns must be 8-aligned");
  CUDA_TRY(mlra::launch_materialize_tile(q->d, row0, nrows, col0, ncols, out, ld,
                                         dtype == MLRA_F32, static_cast<cudaStream_t>(stream)));
  return MLRA_OK;
}

mlra_status mlra_materialize(const mlra_qweight* q, void* out, mlra_dtype dtype, int64_t ld,
                             void* stream) {
  if (mlra_status st = check_q(q)) return st;
  return mlra_materialize_rows(q, 0, q->d.rows, out, dtype, ld, stream);
}

mlra_status mlra_lp_forward(const mlra_qweight* q, mlra_strategy strategy, const void* x,
                            int64_t ldx, int64_t m, void* y, mlra_dtype y_dtype, int64_t ldy,
                            void* stream) {
  return mlra_lp_forward_ex(q, strategy, nullptr, x, ldx, m, y, y_dtype, ldy, stream);
}

mlra_status mlra_lp_forward_ex(const mlra_qweight* q, mlra_strategy strategy,
                               const mlra_hook* hook, const void* x, int64_t ldx, int64_t m,
                               void* y, mlra_dtype y_dtype, int64_t ldy, void* stream) {
  if (mlra_status st = check_q(q)) return st;
  if (m < 0) return fail(MLRA_ERR_DIMENSION, "lp_forward: negative token count");
  if (ldx < q->d.cols)
    return fail(MLRA_ERR_DIMENSION, "lp_forward: input cols %lld != weight cols %lld",
                (long long)ldx, (long long)q->d.cols);
  if (ldy < q->d.rows) return fail(MLRA_ERR_DIMENSION, "lp_forward: output ld < rows");
  if (strategy < MLRA_WEIGHT || strategy > MLRA_MATVEC)
    return fail(MLRA_ERR_CONFIG, "unknown materialization strategy %d", (int)strategy);
  if (mlra_status st = check_device()) return st;
  if (m == 0) return MLRA_OK;
  Scratch sc(static_cast<cudaStream_t>(stream));
  GemmPlan gp{};
  gp.mn = false;
  if (mlra_status st = aligned_act(sc, x, ldx, m, q->d.cols, &gp.act, &gp.ld_act)) return st;
  gp.k_red_valid = q->d.cols;
  gp.tokens = m;
  gp.out = y;
  gp.ldo = ldy;
  gp.out_f32 = y_dtype == MLRA_F32;
  return run_gemm(q, strategy, hook, gp, sc);
}

mlra_status mlra_lp_backward(const mlra_qweight* q, mlra_strategy strategy, const void* g,
                             int64_t ldg, int64_t m, void* dx, mlra_dtype dx_dtype,
                             int64_t lddx, void* stream) {
  return mlra_lp_backward_ex(q, strategy, nullptr, g, ldg, m, dx, dx_dtype, lddx, stream);
}

mlra_status mlra_lp_backward_ex(const mlra_qweight* q, mlra_strategy strategy,
                                const mlra_hook* hook, const void* g, int64_t ldg, int64_t m,
                                void* dx, mlra_dtype dx_dtype, int64_t lddx, void* stream) {
  if (mlra_status st = check_q(q)) return st;
  if (m < 0) return fail(MLRA_ERR_DIMENSION, "lp_backward: negative token count");
  if (ldg < q->d.rows)
    return fail(MLRA_ERR_DIMENSION, "lp_backward: grad cols %lld != weight rows %lld",
                (long long)ldg, (long long)q->d.rows);
  if (lddx < q->d.cols) return fail(MLRA_ERR_DIMENSION, "lp_backward: output ld < cols");
  if (strategy < MLRA_WEIGHT || strategy > MLRA_MATVEC)
    return fail(MLRA_ERR_CONFIG, "unknown materialization strategy %d", (int)strategy);
  if (mlra_status st = check_device()) return st;
  if (m == 0) return MLRA_OK;
  Scratch sc(static_cast<cudaStream_t>(stream));
  GemmPlan gp{};
  gp.mn = true;
  if (mlra_status st = aligned_act(sc, g, ldg, m, q->d.rows, &gp.act, &gp.ld_act)) return st;
  gp.k_red_valid = q->d.rows;
  gp.tokens = m;
  gp.out = dx;
  gp.ldo = lddx;
  gp.out_f32 = dx_dtype == MLRA_F32;
  return run_gemm(q, strategy, hook, gp, sc);
}

mlra_status mlra_lora_forward(const mlra_lora* L, const void* x, int64_t ldx, int64_t m, void* y,
                              mlra_dtype y_dtype, int64_t ldy, float* xb, void* stream) {
  ProfScope call_scope(3);
  if (mlra_status st = check_lora(L)) return st;
  const QWeightDev& d = L->q->d;
  if (m < 0) return fail(MLRA_ERR_DIMENSION, "layer: negative token count");
  if (ldx < d.cols)
    return fail(MLRA_ERR_DIMENSION, "layer: input cols %lld != d_in %lld", (long long)ldx,
                (long long)d.cols);
  if (ldy < d.rows) return fail(MLRA_ERR_DIMENSION, "layer: output ld < d_out");
  if (!xb) return fail(MLRA_ERR_CONTRACT, "layer: xb buffer required (saved for backward)");
  if (mlra_status st = check_device()) return st;
  if (m == 0) return MLRA_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Scratch sc(s);
  const int64_t r = L->rank, rp = round_up(r, 64);
  const float scaling = static_cast<float>(L->alpha / static_cast<double>(r));
  GemmPlan gp{};
  gp.mn = false;
  if (mlra_status st = aligned_act(sc, x, ldx, m, d.cols, &gp.act, &gp.ld_act)) return st;
  auto* xbs = sc.get<__nv_bfloat16>(static_cast<size_t>(m * rp));
  auto* apad = sc.get<__nv_bfloat16>(static_cast<size_t>(d.rows_pad * rp));
  if (!xbs || !apad) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  mlra::PrepBatch pb;
  pb.pad(L->a, d.rows, r, r, 1.0f, apad, d.rows_pad, rp);  // A -> padded bf16 GEMM operand
  unsigned* flags = gemm_flags(sc, pb);
  if (!flags) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  // K4: xb = x·B (matmul(t, x, B), lora.cpp:68), finished with bf16(s·xb) zero
  // padded to rp columns: the extra-K LoRA operand of the GEMM
  if (mlra::thin_fused_ok(r, m)) {
    // one launch: B is split in the kernel, A's padded operand and the flags
    // are the launch's post jobs (no prep launch in front of it)
    mlra::ThinOut o;
    o.out = xb;
    o.ldo = r;
    o.pad = xbs;
    o.ldp = rp;
    o.pad_cols = static_cast<int>(rp);
    o.pad_scale = scaling;
    o.trace = thin_trace();
    CUDA_TRY(mlra::launch_rowmma_fused(gp.act, gp.ld_act, m, d.cols, L->b, r, r, o, pb, s));
  } else {
    // prep launch: B -> transposed hi/lo planes, A's operand, counters = 0
    Planes bt;
    ThinWs tw;
    if (mlra_status st = make_planes(sc, pb, L->b, d.cols, r, false, &bt)) return st;
    if (mlra_status st = thin_ws(sc, pb, true, m, d.cols, r, false, &tw)) return st;
    CUDA_TRY(mlra::launch_prep(pb, s));
    if (mlra_status st = rows_product(s, tw, gp.act, gp.ld_act, m, d.cols, bt, xb, r, xbs, rp,
                                      scaling, nullptr))
      return st;
  }
  gp.k_red_valid = d.cols;
  gp.act_lora = xbs;
  gp.w_lora = apad;
  gp.rp = rp;
  gp.rank = r;
  gp.tokens = m;
  gp.out = y;
  gp.ldo = ldy;
  gp.out_f32 = y_dtype == MLRA_F32;
  gp.bias = L->bias;
  gp.sk_flags_zeroed = flags;
  // K2: y = x·Ŵᵀ + (s·xb)·Aᵀ + bias
  return run_gemm(L->q, L->strategy, L->hook, gp, sc);
}

mlra_status mlra_lora_backward(const mlra_lora* L, const void* x, int64_t ldx, const float* xb,
                               const void* dy, int64_t lddy, int64_t m, void* dx,
                               mlra_dtype dx_dtype, int64_t lddx, float* da, float* db,
                               float* dbias, void* stream) {
  ProfScope call_scope(3);
  if (mlra_status st = check_lora(L)) return st;
  const QWeightDev& d = L->q->d;
  if (m < 0) return fail(MLRA_ERR_DIMENSION, "layer: negative token count");
  if (ldx < d.cols) return fail(MLRA_ERR_DIMENSION, "layer: input ld < d_in");
  if (lddy < d.rows)
    return fail(MLRA_ERR_DIMENSION, "lp_backward: grad cols %lld != weight rows %lld",
                (long long)lddy, (long long)d.rows);
  if (dx && lddx < d.cols) return fail(MLRA_ERR_DIMENSION, "layer: dx ld < d_in");
  if (!xb || !da || !db) return fail(MLRA_ERR_CONTRACT, "layer: xb/dA/dB buffers required");
  if (mlra_status st = check_device()) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t r = L->rank, rp = round_up(r, 64);
  if (m == 0) {
    CUDA_TRY(cudaMemsetAsync(da, 0, d.rows * r * 4, s));
    CUDA_TRY(cudaMemsetAsync(db, 0, d.cols * r * 4, s));
    if (dbias) CUDA_TRY(cudaMemsetAsync(dbias, 0, d.rows * 4, s));
    return MLRA_OK;
  }
  Scratch sc(s);
  const float scaling = static_cast<float>(L->alpha / static_cast<double>(r));
  const __nv_bfloat16 *xa, *dya;
  int64_t ldxa, lddya;
  if (mlra_status st = aligned_act(sc, x, ldx, m, d.cols, &xa, &ldxa)) return st;
  if (mlra_status st = aligned_act(sc, dy, lddy, m, d.rows, &dya, &lddya)) return st;
  auto* dyA = sc.get<float>(static_cast<size_t>(m * r));
  auto* dyas = sc.get<__nv_bfloat16>(static_cast<size_t>(m * rp));
  auto* bpad = dx ? sc.get<__nv_bfloat16>(static_cast<size_t>(d.cols_pad * rp)) : nullptr;
  if (!dyA || !dyas || (dx && !bpad)) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  // A, xb -> transposed hi/lo planes, B -> the dX GEMM's padded operand, counters = 0
  // (dA, dB, dbias, dyA are stored by the skinny kernels' finishers: no zero-fill).
  // Fused row product (r <= 64): A is split inside it and B's operand and the
  // flags are its post jobs; the planes of xb and the column products' counters
  // (the side stream's inputs) are a prep launch on the side stream.
  const bool fused = mlra::thin_fused_ok(r, m);
  mlra::PrepBatch pb, pbs;  // pb: main stream (prep launch or the row kernel's post jobs)
  Planes at, xbt, dyat;
  ThinWs w_row, w_da, w_db;
  mlra::PrepBatch& cpb = fused ? pbs : pb;  // column-product inputs
  if (mlra_status st = make_planes(sc, cpb, xb, m, r, dbias != nullptr, &xbt)) return st;
  if (mlra_status st = alloc_planes(sc, m, r, false, &dyat)) return st;
  if (mlra_status st = thin_ws(sc, cpb, false, m, d.rows, r, dbias != nullptr, &w_da)) return st;
  if (mlra_status st = thin_ws(sc, cpb, false, m, d.cols, r, false, &w_db)) return st;
  if (dx) pb.pad(L->b, d.cols, r, r, 1.0f, bpad, d.cols_pad, rp);
  if (!fused) {
    if (mlra_status st = make_planes(sc, pb, L->a, d.rows, r, false, &at)) return st;
    if (mlra_status st = thin_ws(sc, pb, true, m, d.rows, r, false, &w_row)) return st;
  }
  unsigned* flags = gemm_flags(sc, pb);
  if (!flags) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  if (!fused) CUDA_TRY(mlra::launch_prep(pb, s));
  // dA early: the side stream starts dA = s·dyᵀ·xb right after the prep launch,
  // concurrently with dY·A — both stream dY, so the second reader finds much of
  // it in L2; dB follows once dYA exists (cfg2 step 1166 -> 1139 us, cfg3 -2 %;
  // MLRA_DA_EARLY=0: dA after dY·A, for A/B)
  static const bool da_early = getenv("MLRA_DA_EARLY") == nullptr || atoi(getenv("MLRA_DA_EARLY")) != 0;
  SideStream* side = nullptr;
  static const bool no_side = getenv("MLRA_NO_SIDE") != nullptr;        // dev A/B switch
  static const bool side_first = getenv("MLRA_SIDE_FIRST") != nullptr;  // dev A/B switch
  if (dx && !no_side) {
    if (mlra_status st = side_stream(&side)) return st;
    CUDA_TRY(cudaEventRecord(side->fork, s));
    CUDA_TRY(cudaStreamWaitEvent(side->st, side->fork, 0));
  }
  if (fused) CUDA_TRY(mlra::launch_prep(pbs, side ? side->st : s));
  const bool early = side != nullptr && da_early;
  auto grad_a = [&](cudaStream_t cs) -> mlra_status {
    // K5b: dA = s·dyᵀ·xb (+ dbias = Σ_t dy)   (autodiff.cpp:153-155, 315-320, 183-191)
    return cols_product(cs, w_da, dya, lddya, m, d.rows, xbt, scaling, da, r, dbias);
  };
  if (early) {
    if (mlra_status st = grad_a(side->st)) return st;
  }
  // K5a: dyA = dy·A ; d(xb) = s·dyA (autodiff.cpp:150-152 on record lora.cpp:69),
  // finished with bf16(s·dyA) (the dX GEMM's extra-K operand) and dyA's
  // transposed hi/lo planes (the dB product's factor)
  if (fused) {
    mlra::ThinOut o;
    o.out = dyA;
    o.ldo = r;
    o.pad = dyas;
    o.ldp = rp;
    o.pad_cols = static_cast<int>(rp);
    o.pad_scale = scaling;
    o.thi = dyat.hi[0];
    o.ldt = dyat.ldt;
    o.t_rows = static_cast<int>(dyat.rows_t[0]);
    o.trace = thin_trace();
    CUDA_TRY(mlra::launch_rowmma_fused(dya, lddya, m, d.rows, L->a, r, r, o, pb, s));
  } else if (mlra_status st = rows_product(s, w_row, dya, lddya, m, d.rows, at, dyA, r, dyas, rp,
                                           scaling, &dyat)) {
    return st;
  }
  // K5b / K6 go to the side stream when a dX GEMM follows, else inline. The GEMM is
  // enqueued FIRST: its persistent pairs take the SMs, and dA / dB fill the SMs
  // its under-filled last wave leaves idle (e.g. 128 tiles over 74 pairs) and its
  // tail, instead of delaying its start (MLRA_SIDE_FIRST=1: the old order).
  if (early) {  // dB needs dYA: the side stream waits for the row product
    CUDA_TRY(cudaEventRecord(side->mid, s));
    CUDA_TRY(cudaStreamWaitEvent(side->st, side->mid, 0));
  }
  auto adapter_grads = [&](cudaStream_t cs) -> mlra_status {
    if (!early) {
      if (mlra_status st = grad_a(cs)) return st;
    }
    // K6: dB = s·xᵀ·dyA   (autodiff.cpp:153-155 on record lora.cpp:68)
    return cols_product(cs, w_db, xa, ldxa, m, d.cols, dyat, scaling, db, r, nullptr);
  };
  if (!dx) return adapter_grads(s);  // frozen input: no dX (autodiff.cpp:136)
  if (!side) {
    if (mlra_status st = adapter_grads(s)) return st;
  } else if (side_first) {
    if (mlra_status st = adapter_grads(side->st)) return st;
  }
  GemmPlan gp{};
  gp.mn = true;
  gp.act = dya;
  gp.ld_act = lddya;
  gp.k_red_valid = d.rows;
  gp.act_lora = dyas;
  gp.w_lora = bpad;
  gp.rp = rp;
  gp.rank = r;
  gp.tokens = m;
  gp.out = dx;
  gp.ldo = lddx;
  gp.out_f32 = dx_dtype == MLRA_F32;
  gp.sk_flags_zeroed = flags;
  gp.no_pdl = side != nullptr;
  // K3: dx = dy·Ŵ + (s·dyA)·Bᵀ   (lp_backward + matmul-bwd dx, lora.cpp:68)
  const mlra_status gst = run_gemm(L->q, L->strategy, L->hook, gp, sc);
  if (side) {
    if (!side_first && gst == MLRA_OK) {
      if (mlra_status st = adapter_grads(side->st)) return st;
    }
    // join: the caller's stream (and the scratch frees queued on it) waits for dA/dB
    CUDA_TRY(cudaEventRecord(side->join, side->st));
    CUDA_TRY(cudaStreamWaitEvent(s, side->join, 0));
  }
  return gst;
}

mlra_status mlra_rht(const void* in, int64_t rows, int64_t cols, int64_t ld_in, const float* signs,
                     int inverse, int block, void* out, int64_t ld_out, mlra_dtype out_dtype,
                     void* stream) {
  if (!in || !out || !signs) return fail(MLRA_ERR_CONTRACT, "rht: null buffers");
  if (block != 64 && block != 128 && block != 256 && block != 512 && block != 1024)
    return fail(MLRA_ERR_CONFIG, "rht: block %d must be a power of two in [64, 1024]", block);
  if (rows < 0 || cols <= 0 || cols % block != 0)
    return fail(MLRA_ERR_DIMENSION, "rht: cols %lld is not a multiple of the block %d",
                (long long)cols, block);
  if (ld_in < cols || ld_out < cols || ld_in % 2 || ld_out % 2 ||
      reinterpret_cast<uintptr_t>(in) % 4 || reinterpret_cast<uintptr_t>(out) % 8)
    return fail(MLRA_ERR_DIMENSION, "rht: leading dimensions / alignment");
  if (out_dtype != MLRA_BF16 && out_dtype != MLRA_F32) return fail(MLRA_ERR_CONFIG, "rht: bad dtype");
  if (mlra_status st = check_device()) return st;
  CUDA_TRY(mlra::launch_rht(in, rows, cols, ld_in, signs, inverse, block, out, ld_out,
                            out_dtype == MLRA_F32, static_cast<cudaStream_t>(stream)));
  return MLRA_OK;
}

mlra_status mlra_adamw_step(const mlra_adamw* opt, int64_t step_index, double lr,
                            int64_t n_params, const int64_t* offsets, double* params, double* m,
                            double* v, const void* grad, mlra_dtype grad_dtype, float* params_f32,
                            int* first_bad, void* stream) {
  if (!opt) return fail(MLRA_ERR_CONTRACT, "adamw: null optimizer config");
  if (n_params < 0 || (n_params > 0 && !offsets))
    return fail(MLRA_ERR_CONTRACT, "adamw: params/names size mismatch");
  if (step_index < 0) return fail(MLRA_ERR_CONTRACT, "adamw: negative step index");
  if (grad_dtype != MLRA_F32 && grad_dtype != MLRA_F64)
    return fail(MLRA_ERR_CONFIG, "adamw: gradients must be f32 or f64");
  if (n_params == 0) return MLRA_OK;
  if (offsets[0] != 0) return fail(MLRA_ERR_CONTRACT, "adamw: offsets[0] must be 0");
  for (int64_t i = 0; i < n_params; ++i)
    if (offsets[i + 1] < offsets[i])
      return fail(MLRA_ERR_CONTRACT, "adamw: offsets must be non-decreasing");
  const int64_t n = offsets[n_params];
  if (n > 0 && (!params || !m || !v || !grad))
    return fail(MLRA_ERR_CONTRACT, "adamw: gradient missing for parameter buffers");
  if (n_params > mlra::kAdamwMaxSegs)
    return fail(MLRA_ERR_CONFIG, "adamw: %lld parameters in one bucket (max %d)",
                (long long)n_params, mlra::kAdamwMaxSegs);
  if (mlra_status st = check_device()) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  // train.cpp:99-101 and the per-element constants of :122-127, on the host
  const double t = static_cast<double>(step_index) + 1.0;
  mlra::AdamwConsts c{};
  c.beta1 = opt->beta1;
  c.one_m_beta1 = 1.0 - opt->beta1;
  c.beta2 = opt->beta2;
  c.one_m_beta2 = 1.0 - opt->beta2;
  c.bc1 = 1.0 - std::pow(opt->beta1, t);
  c.bc2 = 1.0 - std::pow(opt->beta2, t);
  c.lr = lr;
  c.eps = opt->eps;
  c.decay = 1.0 - lr * opt->weight_decay;
  Scratch sc(s);
  int* bad = first_bad ? first_bad : sc.get<int>(1);
  if (!bad) return fail(MLRA_ERR_CUDA, "workspace allocation failed");
  const int nseg = static_cast<int>(n_params);
  static thread_local mlra::AdamwSegs segs;
  for (int64_t i = 0; i <= n_params; ++i) segs.off[i] = offsets[i];
  CUDA_TRY(mlra::launch_adamw(grad, grad_dtype == MLRA_F64, n, segs, nseg, bad, params, m, v,
                              params_f32, c, s));
  if (first_bad) return MLRA_OK;
  int host_bad = nseg;
  CUDA_TRY(cudaMemcpyAsync(&host_bad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  if (host_bad >= 0 && host_bad < nseg)
    return fail(MLRA_ERR_NUMERIC, "adamw: non-finite gradient for parameter #%d at step %lld",
                host_bad, (long long)step_index);
  return MLRA_OK;
}

}  // extern "C"
