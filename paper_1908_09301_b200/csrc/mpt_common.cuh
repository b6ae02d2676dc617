// Shared definitions for the multiple-precision Taylor kernels (sm_100a).
//
// Number format: a value is X * 2^-F with F = 28*Lf and
// X = sum_{j=0..Lf} d_j B^j, B = 2^28, signed digits |d_j| < B that all carry
// the sign of X (canonical sign-magnitude). The Taylor coefficients are
// tau-scaled (a~_i = a_i tau^i) so the step update is an exact sum.
#pragma once
#include <cstdint>

namespace mpt {

constexpr int kRadixBits = 28;
constexpr int64_t kRadix = int64_t(1) << kRadixBits;
constexpr int64_t kMask = kRadix - 1;
constexpr int kR = 8;            // columns per thread group (register window)
constexpr int kPad = 16;         // zero digits on each side of a staged row
constexpr int kMaxD = 4;         // state dimension supported on the device
constexpr int kMaxP = 8;         // distinct product pairs
constexpr int kMaxT = 24;        // bilinear terms
constexpr int kMaxLanesDigits = 24;  // per-lane digits in warp normalisation => ncols <= 768
constexpr int kFoldEvery = 120;  // products per column between carry folds (< 128)

enum Status : int32_t {
  kOk = 0,
  kOverflow = 1,   // a value left the fixed-point range
};

struct Params {
  int D, NT, NP;     // dims, bilinear terms, distinct pairs
  int Lf, W, RS;     // fractional digits, digits per value (Lf+1), row stride (>= W, mult of 4)
  int sc;            // extra digits of the c_i = tau/(i+1) table
  int N;             // Taylor order
  int P;             // reference precision in bits (state rounding)
  int pj[kMaxP], pk[kMaxP];
  int teq[kMaxT], tpair[kMaxT];
  int nlv, nrv;               // distinct left / right variables of the pairs
  int lvar[kMaxP], rvar[kMaxP];
  int pl[kMaxP], pr[kMaxP];   // pair -> index into lvar / rvar
  // bilinear coefficients that are small integers are applied to the exact
  // Cauchy column sums (no intermediate rounding); pairs used by any other
  // term are rounded first (oracle/fixmodel.c small_int)
  int tq_small[kMaxT], tq_int[kMaxT];
  int pair_round[kMaxP];
  int all_q_small;
  int tg_used[kMaxP + kMaxD];  // exchange targets with producers (pair sums, non-integer linear rows)
  int lin_small[kMaxD * kMaxD], lin_int[kMaxD * kMaxD];
  // constants (global, row stride RS)
  const int32_t* cst;   // D rows
  const int32_t* lin;   // D*D rows
  const int32_t* q;     // NT rows
  const int32_t* ctab;  // N rows
  // per-trajectory state
  int n_traj;
  int32_t* coef;        // n_traj * D * (N+1) * RS
  int2* rinfo;          // n_traj * D * (N+1)  (bot, top) of nonzero digits
  int32_t* state;       // n_traj * D * RS (in: initial, out: final)
  int32_t* rec;         // record slots * n_traj * D * RS
  int32_t* status;      // n_traj
  int n_steps, start_step, stride;
  int kc;               // k values staged per chunk
  int nthreads;
  int team_mb;          // team kernel: CTAs per SM (1 or 2; ensembles)
  unsigned long long* counters;  // optional: [0] useful limb-MACs, [1] executed limb-MACs
  int write_coef;                // cluster kernel: also store every coefficient row to `coef`
  long long* dbg;                // debug dump (nullptr in production)
  void* gscratch;                // grid kernel: global accumulators + barrier words
};

}  // namespace mpt
