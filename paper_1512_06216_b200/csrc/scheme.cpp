// SACP cost rule (Alg. 3; costs P:L333 and P:L335) and the shard
// map of a PS layer (reading Z11).  Pure host integer code: no context, no GPU.
#include <algorithm>
#include <limits>

#include "internal.h"

namespace {

bool mul_u64(uint64_t a, uint64_t b, uint64_t* out) { return !__builtin_mul_overflow(a, b, out); }
bool add_u64(uint64_t a, uint64_t b, uint64_t* out) { return !__builtin_add_overflow(a, b, out); }

}  // namespace

extern "C" int32_t poseidon_choose_scheme(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P,
                                          poseidon_costs_t* costs) {
  using namespace poseidon;
  if (M < 0 || N < 0 || K < 0 || P < 1) {
    fail(POSEIDON_ERR_INVALID_ARG, "choose_scheme: need M, N, K >= 0 and P >= 1");
    return POSEIDON_ERR_INVALID_ARG;
  }
  const uint64_t m = (uint64_t)M, n = (uint64_t)N, k = (uint64_t)K, p = (uint64_t)P;
  uint64_t mpn, pm1sq, sfb, pk, pkmn, pmn, sfps, full;
  // C_sfb = (P-1)^2 K (M+N)
  bool ok = add_u64(m, n, &mpn) && mul_u64(p - 1, p - 1, &pm1sq) && mul_u64(pm1sq, k, &sfb) &&
            mul_u64(sfb, mpn, &sfb);
  // C_sfps = P K (M+N) + P M N
  ok = ok && mul_u64(p, k, &pk) && mul_u64(pk, mpn, &pkmn) && mul_u64(p, m, &pmn) && mul_u64(pmn, n, &pmn) &&
       add_u64(pkmn, pmn, &sfps);
  // C_full = 2 P M N
  ok = ok && mul_u64(2, pmn, &full);
  if (!ok) {
    fail(POSEIDON_ERR_INVALID_ARG, "choose_scheme: cost overflows 64 bits");
    return POSEIDON_ERR_INVALID_ARG;
  }
  if (costs) {
    costs->sfb = sfb;
    costs->sf_ps = sfps;
    costs->full_ps = full;
  }
  if (kind != POSEIDON_LAYER_FC) return POSEIDON_SCHEME_PS;       // Alg. 3 lines 1-3
  return sfb <= sfps ? POSEIDON_SCHEME_SFB : POSEIDON_SCHEME_PS;   // Alg. 3 line 5, tie -> SFB
}

extern "C" poseidon_status_t poseidon_shard_range(int64_t n, int32_t P, int32_t rank, int64_t* begin,
                                                  int64_t* end, int64_t* padded_n) {
  using namespace poseidon;
  if (n < 0 || P < 1 || rank < 0 || rank >= P)
    return fail(POSEIDON_ERR_INVALID_ARG, "shard_range: need n >= 0, P >= 1, 0 <= rank < P");
  const int64_t A = 32;
  const int64_t S = A * ((n + A * P - 1) / (A * P));
  const int64_t b = rank * S < n ? rank * S : n;
  const int64_t e = (rank + 1) * S < n ? (rank + 1) * S : n;
  if (begin) *begin = b;
  if (end) *end = e;
  if (padded_n) *padded_n = S * P;
  return POSEIDON_OK;
}

// Measured-cost SACP variant: the paper's rule counts floats on Ethernet, where
// reconstruction is "often negligible compared to communication".  On NVLink it is not, so
// this alpha-beta + roofline model of the two B200 executions is reported BESIDE the paper's rule
// (the rule stays the default and is bit-exact); see profiles/c5_crossover_r1.md for measurements.
extern "C" int32_t poseidon_choose_scheme_model(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P,
                                                const poseidon_hw_t* hw, double* t_sfb_us, double* t_ps_us) {
  using namespace poseidon;
  if (M < 0 || N < 0 || K < 0 || P < 1 || !hw || hw->nvlink_gbps <= 0 || hw->hbm_gbps <= 0 ||
      hw->tensor_tflops <= 0) {
    fail(POSEIDON_ERR_INVALID_ARG, "choose_scheme_model: bad arguments");
    return POSEIDON_ERR_INVALID_ARG;
  }
  const double m = (double)M, n = (double)N, k = (double)K, p = (double)P;
  const double nvl = hw->nvlink_gbps * 1e9, hbm = hw->hbm_gbps * 1e9, tc = hw->tensor_tflops * 1e12;
  const double alpha = hw->collective_latency_us * 1e-6;
  const double ldk = 4.0 * ((K + 3) / 4);
  // SFB: pack (read + write both factors) + all-gather of everyone's factors + K1
  const double t_pack = 8.0 * k * (m + n) / hbm;
  const double t_ag = (P > 1) ? ((p - 1.0) * ldk * (m + n) * 4.0 / nvl + alpha) : 0.0;
  const double t_k1 = std::max(2.0 * m * n * p * k / tc, (8.0 * m * n + 4.0 * p * ldk * (m + n)) / hbm);
  const double t_sfb = t_pack + t_ag + t_k1;
  // PS: local dW GEMM (which SFB skips) + reduce-scatter + K2 + all-gather
  const double t_wgrad = std::max(2.0 * m * n * k / tc, (4.0 * k * (m + n) + 4.0 * m * n) / hbm);
  const double t_rsag = (P > 1) ? (2.0 * (p - 1.0) / p * 4.0 * m * n / nvl + 2.0 * alpha) : 0.0;
  const double t_k2 = 12.0 * m * n / p / hbm;
  const double t_ps = t_wgrad + t_rsag + t_k2;
  if (t_sfb_us) *t_sfb_us = t_sfb * 1e6;
  if (t_ps_us) *t_ps_us = t_ps * 1e6;
  if (kind != POSEIDON_LAYER_FC) return POSEIDON_SCHEME_PS;
  return t_sfb <= t_ps ? POSEIDON_SCHEME_SFB : POSEIDON_SCHEME_PS;
}

// The same model with the literal else-branch of Alg. 3 as a third execution (SF-PS, reading Z20):
// pack + V all-gather + U rows to their masters + K1 on the master's R = 32-aligned ceil(M/P) rows + the
// masters' rows pushed to everyone.  Returns 0 (PS), 1 (SFB) or 2 (SF-PS), whichever is predicted fastest
// (non-FC -> PS); reported beside the rule (profiles/sfps_crossover_r1.md for the measurements).
extern "C" int32_t poseidon_choose_scheme_model3(int32_t kind, int64_t M, int64_t N, int64_t K, int32_t P,
                                                 const poseidon_hw_t* hw, double* t_sfb_us, double* t_ps_us,
                                                 double* t_sfps_us) {
  using namespace poseidon;
  double ts = 0.0, tp = 0.0;
  const int32_t two = poseidon_choose_scheme_model(kind, M, N, K, P, hw, &ts, &tp);
  if (two < 0) return two;
  const double m = (double)M, n = (double)N, k = (double)K, p = (double)P;
  const double nvl = hw->nvlink_gbps * 1e9, hbm = hw->hbm_gbps * 1e9, tc = hw->tensor_tflops * 1e12;
  const double alpha = hw->collective_latency_us * 1e-6;
  const double ldk = 4.0 * ((K + 3) / 4);
  int64_t b0 = 0, e0 = 0, pad = 0;
  poseidon_shard_range(M, P, 0, &b0, &e0, &pad);
  const double r = (double)(e0 - b0);   // the largest master's rows (rank 0 owns a full shard)
  const double t_pack = 8.0 * k * (m + n) / hbm;
  const double t_comm = (P > 1) ? ((p - 1.0) * ldk * n * 4.0 / nvl + (p - 1.0) * ldk * r * 4.0 / nvl +
                                   (m - r) * n * 4.0 / nvl + 3.0 * alpha)
                                : 0.0;
  const double t_k1 = std::max(2.0 * r * n * p * k / tc, (8.0 * r * n + 4.0 * p * ldk * (r + n)) / hbm);
  const double tf = t_pack + t_comm + t_k1;
  if (t_sfb_us) *t_sfb_us = ts;
  if (t_ps_us) *t_ps_us = tp;
  if (t_sfps_us) *t_sfps_us = tf * 1e6;
  if (kind != POSEIDON_LAYER_FC) return POSEIDON_SCHEME_PS;
  const double best2 = std::min(ts, tp);
  if (tf * 1e6 < best2) return POSEIDON_SCHEME_SFPS;
  return two;
}
