// qgemm2.cu — host side of the CTA-pair kernel (qgemm2_kernel.cuh): the
// schedule planner (whole tiles / stream-K / split-K), the kernel choice cost
// model, and the launch dispatch onto the four per-family translation units.
#include "qgemm2_kernel.cuh"

namespace mlra {

namespace {

constexpr double kSkMinIdleBlocks = 50.0;  // stream-K only when it recovers more than this
constexpr int64_t kSkMinBlocksPerPair = 8;
constexpr int64_t kSplitMinBlocks = 8;  // split-K: k-blocks per pair at least
#ifndef MLRA_SPLIT_FIX
#define MLRA_SPLIT_FIX 16.0
#endif
// split-K: moving one whole 512-token accumulator (256 KB per CTA) out and in
constexpr double kSplitFixUnits = MLRA_SPLIT_FIX;
constexpr double kSplitSync = 3.0;  // publish / acquire / first slab latency
#ifndef MLRA_COST_TOK256
#define MLRA_COST_TOK256 0.7
#endif
constexpr double kCostTok256 = MLRA_COST_TOK256;  // 256-token pair k-block, pair units
constexpr double kSkFixUnits = 56.0;  // stream-K partial write + in-order owner fix-up
constexpr double kSkMaxWaves = 1.25;  // stream-K only below this many waves of whole tiles
#ifndef MLRA_COST128
#define MLRA_COST128 0.85
#endif
constexpr double kCost128 = MLRA_COST128;  // 1-CTA 128-token k-block wave, pair units
constexpr double kCost256 = 0.8;           // 1-CTA 256-token k-block wave, pair units

}  // namespace


namespace {

// Split-K schedule: every pair one (tile, k-range) unit, tiles of 512 or 256
// tokens (tok256: one accumulator), S pairs per tile.
void set_split(GemmArgs& p, int64_t tiles, int64_t S, int64_t n_kb, bool tok256) {
  (void)n_kb;  // pair q: tile q / S, k-blocks from n_kb * (q % S) / S (sk_cut)
  p.sk_pairs = static_cast<int>(tiles * S);
  p.split = static_cast<int>(S);
  p.tok256 = tok256 ? 1 : 0;
}

// Plans the schedule and returns its modelled cost in pair-k-block units (a
// 512-token pair k-block ~0.75 us). Candidates: whole 512-token tiles strided
// over the pairs; split-K over 512- or 256-token tiles (one wave, S ways, S = 1
// allowed for 256: whole half-width tiles); stream-K (under-filled last wave).
// The split fix-up moves (S-1)/S of every CTA's accumulator through L2 (~32 B
// per clock per SM each way: 256 KB ~ kSplitFixUnits), so half-width tiles
// halve it at the price of less weight reuse per MMA (kCostTok256 per k-block).
double plan_pair(GemmArgs& p) {
  p.sk_pairs = 0;
  p.split = 0;
  p.tok256 = 0;
  const int64_t tiles = (p.m_total / PAIR_ROWS) * ((p.tokens + PAIR_TOK - 1) / PAIR_TOK);
  const int64_t tiles256 = (p.m_total / PAIR_ROWS) * ((p.tokens + PAIR_TOK / 2 - 1) / (PAIR_TOK / 2));
  const int64_t n_kb = p.n_kb_main + p.n_kb_lora;
  int64_t slots = sm_total() / 2;
  if (slots > kMaxSkPairs) slots = kMaxSkPairs;
  // MLRA_SK=0: whole tiles; 1: stream-K; 4 / 5: split-K on 512 / 256-token
  // tiles; default (2): the cheapest by the cost model
  int mode = 2;
  if (const char* e = getenv("MLRA_SK")) mode = atoi(e);
  const int64_t waves = tiles > 0 ? (tiles + slots - 1) / slots : 0;
  const double whole = static_cast<double>(waves) * static_cast<double>(n_kb);
  if (mode == 0 || tiles <= 0) return whole;
  auto split_cost = [&](int64_t t, int64_t S, bool half) {
    const double kb = static_cast<double>(n_kb) / static_cast<double>(S);
    const double fix = S > 1 ? kSplitFixUnits * (half ? 0.5 : 1.0) *
                                   static_cast<double>(S - 1) / static_cast<double>(S) + kSplitSync
                             : 0.0;
    (void)t;
    return kb * (half ? kCostTok256 : 1.0) + fix;
  };
  auto max_ways = [&](int64_t t, bool half) {
    int64_t S = slots / t;
    if (S > n_kb / kSplitMinBlocks) S = n_kb / kSplitMinBlocks;
    if (S > kSplitMaxS) S = kSplitMaxS;
    if (!half && S < 2) S = 0;
    return S;
  };
  if (mode == 4 || mode == 5) {  // forced split-K (tests, probes)
    const bool half = mode == 5;
    const int64_t t = half ? tiles256 : tiles;
    const int64_t S = t > 0 ? max_ways(t, half) : 0;
    if (S >= 1) {
      set_split(p, t, S, n_kb, half);
      return split_cost(t, S, half);
    }
    return whole;
  }
  // cheapest split-K candidate (one wave of (tile, k-range) units)
  double best = 1e30;
  int64_t best_S = 0;
  bool best_half = false;
  if (mode == 2) {
    for (int h = 0; h < 2; ++h) {
      const bool half = h == 1;
      const int64_t t = half ? tiles256 : tiles;
      for (int64_t S = half ? 1 : 2; S <= max_ways(t, half); ++S) {
        const double c = split_cost(t, S, half);
        if (c < best) {
          best = c;
          best_S = S;
          best_half = half;
        }
      }
    }
  }
  // Stream-K (equal contiguous k-block ranges over the pairs, in-order owner
  // fix-up) replaces whole tiles below ~1.25 waves when the last wave would idle
  // more than ~50 k-blocks per pair (measured: above that, cfg3 5.69 vs 6.18 ms
  // and cfg4 b3 2.37 vs 2.51 ms per step with whole tiles); a cheaper split-K
  // plan beats either.
  const double idle_kb = static_cast<double>(n_kb) *
                         (static_cast<double>(waves) - static_cast<double>(tiles) / slots);
  const bool sk_ok = mode == 1 || (idle_kb >= kSkMinIdleBlocks &&
                                   static_cast<double>(tiles) <= kSkMaxWaves * static_cast<double>(slots));
  if (sk_ok) {
    const int64_t total = tiles * n_kb;
    int64_t pairs = slots;
    if (total / pairs < kSkMinBlocksPerPair) pairs = total / kSkMinBlocksPerPair;
    const double c = pairs >= 2 ? static_cast<double>(total) / pairs + kSkFixUnits : 1e30;
    if (pairs >= 2 && (mode == 1 || c <= best)) {
      // pair q starts at k-block total * q / pairs (sk_cut)
      p.sk_pairs = static_cast<int>(pairs);
      return c;
    }
  }
  if (best_S == 0 || best >= whole) return whole;
  if (best_S > 0) set_split(p, best_half ? tiles256 : tiles, best_S, n_kb, best_half);
  return best;
}

}  // namespace

void qgemm2_plan(GemmArgs& p) { plan_pair(p); }

// Kernel choice for a GEMM of p.tokens tokens (p's tile extents set, schedule
// not yet planned). Costs in pair-k-block-wave units, fitted to graph-timed
// sweeps at the LLaMA-7B shapes (scripts/sk_probe.py): a pair k-block wave
// ~0.8 us, a 1-CTA k-block wave ~0.6-0.7 us (0.8 units) with 256-token tiles
// and ~0.7 us (0.85 units) with 128-token tiles — the 1-CTA MMA is bound by
// shared-memory operand traffic (A 4 KB + B N·32 B per 16-deep step), not by N
// — stream-K's partial write +
// in-order fix-up ~56 units, split-K's distributed fix-up ~kSplitFixUnits.
// Returns 2 (pair), 1 (1-CTA, 256) or 3 (1-CTA, 128).
int qgemm_choose(const GemmArgs& p0) {
  GemmArgs p = p0;
  const double pair0 = plan_pair(p);
  const int64_t sms = sm_total();
  const double n_kb = static_cast<double>(p.n_kb_main + p.n_kb_lora);
  const int64_t tiles1 = (p.m_total / BM) * ((p.tokens + 255) / 256);
  const int64_t tiles3 = (p.m_total / BM) * ((p.tokens + 127) / 128);
  // a whole 512-token pair tile over <= 256 tokens is half empty
  const double pair = (p0.tokens <= 256 && !p.split) ? 1e30 : pair0;
  const double cta1 = static_cast<double>((tiles1 + sms - 1) / sms) * n_kb * kCost256;
  const double cta3 = static_cast<double>((tiles3 + sms - 1) / sms) * n_kb * kCost128;
  if (cta3 < 0.95 * cta1 && cta3 < 0.95 * pair) return 3;
  return cta1 >= 0.95 * pair ? 2 : 1;
}

cudaError_t qgemm2_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                          bool w_tma, bool mn, bool out_f32, cudaStream_t stream) {
  if (p.tokens <= 0 || p.m_total <= 0) return cudaSuccess;
  const bool sk = p.sk_pairs != 0;
  const char* o4 = sk ? getenv("MLRA_SK_OWNER4") : nullptr;  // read per launch, like MLRA_SK
  if (o4 && o4[0] == '1') {
    GemmArgs p4 = p;
    p4.sk_owner4 = 1;
    return mn ? qgemm2_launch_d1(maps, q, p4, w_tma, out_f32, stream)
              : qgemm2_launch_f1(maps, q, p4, w_tma, out_f32, stream);
  }
  if (mn) return sk ? qgemm2_launch_d1(maps, q, p, w_tma, out_f32, stream)
                    : qgemm2_launch_d0(maps, q, p, w_tma, out_f32, stream);
  return sk ? qgemm2_launch_f1(maps, q, p, w_tma, out_f32, stream)
            : qgemm2_launch_f0(maps, q, p, w_tma, out_f32, stream);
}

}  // namespace mlra
