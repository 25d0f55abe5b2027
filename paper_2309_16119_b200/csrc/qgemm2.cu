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
#define MLRA_SPLIT_FIX 24.0
#endif
constexpr double kSplitFixUnits = MLRA_SPLIT_FIX;  // split-K drain + distributed fix-up
constexpr double kSkMaxWaves = 1.25;  // stream-K only below this many waves of whole tiles
#ifndef MLRA_COST128
#define MLRA_COST128 0.85
#endif
constexpr double kCost128 = MLRA_COST128;  // 1-CTA 128-token k-block wave, pair units
constexpr double kCost256 = 0.8;           // 1-CTA 256-token k-block wave, pair units

}  // namespace


void qgemm2_plan(GemmArgs& p) {
  p.sk_pairs = 0;
  p.split = 0;
  const int64_t tiles = (p.m_total / PAIR_ROWS) * ((p.tokens + PAIR_TOK - 1) / PAIR_TOK);
  const int64_t n_kb = p.n_kb_main + p.n_kb_lora;
  int64_t slots = sm_total() / 2;
  if (slots > kMaxSkPairs) slots = kMaxSkPairs;
  int mode = 2;  // MLRA_SK=0: whole tiles; 1: always stream-K; default: when waves quantize
  if (const char* e = getenv("MLRA_SK")) mode = atoi(e);
  if (mode == 0 || tiles <= 0) return;
  // Whole tiles leave n_kb * (waves - tiles/slots) k-blocks of every pair's time
  // idle in the last wave; stream-K pays a roughly fixed fix-up cost (owners
  // read their contributors' partials chunk by chunk at the end). Measured
  // break-even is ~45 k-blocks (m in {512..4096} at LLaMA-7B shapes, all of
  // them at most one wave of tiles).
  const int64_t waves = (tiles + slots - 1) / slots;
  const double idle_kb = static_cast<double>(n_kb) *
                         (static_cast<double>(waves) - static_cast<double>(tiles) / slots);
  if (mode == 2 && idle_kb < kSkMinIdleBlocks) return;
  // With more than ~1.25 waves of whole tiles, splitting every tile across
  // pairs costs more in partial traffic and fix-ups than the last wave's idle
  // time it recovers (measured: cfg3 5.69 vs 6.18 ms, cfg4 b3 2.37 vs 2.51 ms
  // per step with whole tiles), so stream-K is kept for the under-filled cases.
  if (mode == 2 && static_cast<double>(tiles) > kSkMaxWaves * static_cast<double>(slots)) return;
  // every pair needs a few k-blocks of its own, so cuts never collide
  // Split-K (every pair one (tile, k-range) unit, distributed fix-up) when the
  // tiles leave at least half the pairs idle; MLRA_SK=4 forces it, 1 stream-K.
  if (mode != 1) {
    int64_t S = slots / tiles;
    if (S > n_kb / kSplitMinBlocks) S = n_kb / kSplitMinBlocks;
    if (S > 16) S = 16;
    if (S >= 2 && (mode == 4 || 2 * tiles <= slots)) {
      for (int64_t q = 0; q <= tiles * S; ++q) {
        const int64_t t = q / S, sp = q % S;
        int64_t b = n_kb * sp / S;
        if (b & 1) ++b;  // even offset: a Q-ring stage holds two k-blocks
        p.sk_tile[q] = static_cast<int>(t);
        p.sk_off[q] = static_cast<int>(b);
      }
      p.sk_pairs = static_cast<int>(tiles * S);
      p.split = static_cast<int>(S);
      return;
    }
  }
  if (mode == 4) return;
  const int64_t total = tiles * n_kb;
  int64_t pairs = slots;
  if (total / pairs < kSkMinBlocksPerPair) pairs = total / kSkMinBlocksPerPair;
  if (pairs < 2) return;
  for (int64_t q = 0; q <= pairs; ++q) {
    int64_t b = total * q / pairs;
    if ((b % n_kb) & 1) ++b;  // even offset: a Q-ring stage holds two k-blocks
    p.sk_tile[q] = static_cast<int>(b / n_kb);
    p.sk_off[q] = static_cast<int>(b % n_kb);
  }
  p.sk_pairs = static_cast<int>(pairs);
}

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
  qgemm2_plan(p);
  const int64_t sms = sm_total(), slots = sms / 2;
  const double n_kb = static_cast<double>(p.n_kb_main + p.n_kb_lora);
  const int64_t tiles2 = (p.m_total / PAIR_ROWS) * ((p.tokens + PAIR_TOK - 1) / PAIR_TOK);
  const int64_t tiles1 = (p.m_total / BM) * ((p.tokens + 255) / 256);
  const int64_t tiles3 = (p.m_total / BM) * ((p.tokens + 127) / 128);
  const double pair = (p0.tokens <= 256 && !p.split) ? 1e30  // half-empty 512-token tiles
                      : p.sk_pairs ? static_cast<double>(tiles2) * n_kb / p.sk_pairs +
                                         (p.split ? kSplitFixUnits : 56.0)
                                   : static_cast<double>((tiles2 + slots - 1) / slots) * n_kb;
  const double cta1 = static_cast<double>((tiles1 + sms - 1) / sms) * n_kb * kCost256;
  const double cta3 = static_cast<double>((tiles3 + sms - 1) / sms) * n_kb * kCost128;
  if (cta3 < 0.95 * cta1 && cta3 < 0.95 * pair) return 3;
  return cta1 >= 0.95 * pair ? 2 : 1;
}

cudaError_t qgemm2_launch(const GemmMaps& maps, const QWeightDev& q, const GemmArgs& p,
                          bool w_tma, bool mn, bool out_f32, cudaStream_t stream) {
  if (p.tokens <= 0 || p.m_total <= 0) return cudaSuccess;
  const bool sk = p.sk_pairs != 0;
  if (mn) return sk ? qgemm2_launch_d1(maps, q, p, w_tma, out_f32, stream)
                    : qgemm2_launch_d0(maps, q, p, w_tma, out_f32, stream);
  return sk ? qgemm2_launch_f1(maps, q, p, w_tma, out_f32, stream)
            : qgemm2_launch_f0(maps, q, p, w_tma, out_f32, stream);
}

}  // namespace mlra
