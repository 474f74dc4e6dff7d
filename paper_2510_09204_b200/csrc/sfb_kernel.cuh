// sfb_kernel.cuh — persistent per-member SF solve kernel for sm_100a.
//
// One CTA owns one member (instance x sample) for the whole solve; xi, lambda and
// every intermediate stay in shared memory / registers across iterations, HBM sees
// only the warm start, the instance data and the results. One iteration is the map
// of the reference `_step` (pkg/src/swarmplan/solver.py:211-243), computed through
// the exact rewrites of DESIGN.md §3 (oracle/sf_kron.py is the FP64 restatement):
//
//  A  positions   p_i(k) = sum_c W[k,c] xi_i,c in FP64           (constraints.py:159-163)
//  B  screening   FP32 packed (FADD2/FFMA2) r^2 test of every pair / obstacle row of
//                 the lane's robot against a conservative threshold, one bit per body
//                 (funnel-shift accumulation, 2 integer ops per body)
//  B' exact rows  survivors only: FP64 delta, rho = |delta|_scaled, r1 = delta(1 - clip(rho)/rho)
//                 (constraints.py:166-247), accumulated into g_i(k) (= F^T r1 rows)
//  B" box rows    r2 = max(p - p_max, 0) - max(p_min - p, 0) (solver.py:166-168)
//  C  contraction G_i = W^T g_i (= F^T r1 + G^T r2), per-warp partials, fixed-order
//                 cross-warp sum (deterministic, batch-composition independent)
//  D  decision    primal = |r1| + |r2| of the input xi, trace, convergence (solver.py:310-337)
//  E  KKT         lambda+ = lambda - rho G; Delta = 2 lambda+ - lambda + t - Q xi;
//                 xi+ = xi + (I (x) Pxx + 11^T/n (x) (Rxx - Pxx)) Delta + (same xb) (b - A xi)
//
// Thread layout: lanes own robots, a warp owns a k-group (2 consecutive grid steps;
// n <= 16 packs several k-groups per warp). Pair screening loads the partner's FP32
// positions with a warp-broadcast LDS.128; the partner's exact FP64 position comes
// from its owner lane by shuffle (n <= 32) or from FP32 hi/lo pairs in smem (n > 32).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace sfb {

#ifndef SFB_MAXW
#define SFB_MAXW 8
#endif
constexpr int NW = SFB_MAXW;     // max warps per CTA of the default builds (the launch uses P.nw <= NW)
constexpr int NW_RED = 16;       // warp-partial slots in shared memory (the widest build: 16 warps)
constexpr int NBM = 6;           // max boundary rows per robot (rest-to-rest; 2 otherwise)
constexpr int NT = NW * 32;      // max threads per CTA
constexpr float PAD_SMEM = -3.0e30f;   // padded (k >= K1 or dummy body) position in shared memory
constexpr float PAD_OWN = 3.0e30f;     // padded step in the owner's registers -> never a hit
constexpr double COS_HALF_PI = 6.123233995736766e-17;  // cos(pi/2) as the reference evaluates it
constexpr int GRID = 32;         // obstacle candidate grid cells per axis (compact mode)
// per-member constants kept in shared memory instead of registers (read where used, so the
// task loop keeps its registers for the screen): doubles, then floats at KC_F
enum { KC_INV_A2 = 0, KC_INV_B2, KC_RA, KC_RB, KC_DMAX, KC_BLO, KC_BHI = KC_BLO + 3, KC_NDBL = KC_BHI + 3 };
enum { KC_F_BLO = 0, KC_F_BHI = 3, KC_F_GX0 = 6, KC_F_GY0, KC_F_GIX, KC_F_GIY, KC_NFLT };
constexpr int KC_BYTES = KC_NDBL * 8 + KC_NFLT * 4;

struct Layout {       // byte offsets into dynamic shared memory
  int xi, lam, tgt, w, e, q, pxx, pxb, dxx, dxb, g, bv, red, obs_ax, obs_thr, obs_c, obs_s, obs, pmax, gl, uni;
  int grid;           // static-obstacle candidate grid [GRID][GRID] u32 (compact mode)
  int kc;             // per-member constants read at their (rare) use sites: KC_* below
  int ub;             // TBL: boundary rows u [ND*n][NB] + their robot sums [ND][NB]
  int pb;             // TBL: [Pxx | Pxb]^T as DMMA B fragments [k-step][8-column tile][lane]
  int xg;             // cluster exchange buffers [2][nv + 2] (set at launch when csize > 1)
  int uni_bytes, total;
  int slots;          // G partial slots that fit in the union region per round
};

struct KParams {
  int n, m, MP, K1, NB, NKG, RB, obs_static, nw;
  int compact;     // n <= 32, MP <= 32: obstacle candidate grid + FP32 box prescreen (static obstacles)
  int kgs;         // n > 32: k-group position rows held per CTA (2 ring slots per k-group worker)
  int csize;       // CTAs per member (thread-block cluster along the time axis), 1..8
  int mode, max_iters, early_exit;
  double rho, primal_tol, fp_tol, d_max, inv_n;
  float plim;      // FP32 screening valid while max|p| <= plim * (smallest contact axis)
  Layout L;
  const double* consts;
  int B;
  const int* member_instance;
  const double* xi0;
  const double* lam0;
  const double* target;
  const double* bvals;
  const double* box;
  const double* obs_pos;
  const double* obs_axes;
  const double* pair_axes;
  double* xi;
  double* lam;
  double* primal;
  double* eq_max;
  int* iterations;
  int* status;
  double* trace;
  unsigned long long* counters;
  // split schedule (csize == 1, more members than resident CTAs): the grid is one wave of
  // persistent CTAs and CTA c runs evaluation units [c U / G, (c + 1) U / G) of the
  // member-major unit list (U = B (max_iters + 1)); a member cut at a unit boundary is handed
  // from CTA c to CTA c + 1 through hand_flag[c] / hand[c] (and the member's xi / lam outputs)
  int split;
  unsigned* hand_flag;   // [G] 0 = pending, 1 = handed over, 2 = member already finished
  double* hand;          // [G][2 * nt] per-thread fixed-point partial and boundary-residual max
  unsigned jitter_seed;  // race stress build only (SFB_CHECKS): 0 = no perturbation
};

// plan constant block offsets (doubles)
struct ConstOff {
  int W, E, Q, Pxx, Pxb, Dxx, Dxb, total;
  __host__ __device__ static ConstOff make(int K1, int NXI, int NB) {
    ConstOff c;
    c.W = 0;
    c.E = c.W + K1 * NXI;
    c.Q = c.E + NB * NXI;
    c.Pxx = c.Q + NXI * NXI;
    c.Pxb = c.Pxx + NXI * NXI;
    c.Dxx = c.Pxb + NXI * NB;
    c.Dxb = c.Dxx + NXI * NXI;
    c.total = c.Dxb + NXI * NB;
    return c;
  }
};

// shared-memory row stride of xi / lambda: even (16-B aligned rows for LDS.128) and an odd
// number of 16-B units, so 8 lanes loading 8 different rows hit 8 different bank groups
__host__ __device__ constexpr int nxi_pad(int nxi) { return ((nxi + 1) & ~1) % 4 == 0 ? ((nxi + 1) & ~1) + 2 : ((nxi + 1) & ~1); }

// row stride (doubles) of the g table: cols rounded up to 16; column c of row k is stored at
// c ^ tab_swz(k), so a half-warp's DMMA B fragment load (4 k-rows x 4 consecutive columns)
// hits 16 distinct bank pairs without row padding
__host__ __device__ constexpr int tab_stride(int cols) { return (cols + 15) & ~15; }
__host__ __device__ constexpr int tab_swz(int k) { return (k & 3) << 2; }
// W in shared memory: rows of WSTR = 12 doubles (n_basis <= 12, zero padded), all 2 * NKG
// steps rounded up to 4. Rows 96 B apart: the 4 k-rows x 4 columns of a half-warp's DMMA A
// fragment load hit 16 distinct bank pairs, and a task's two step rows load as double2 pairs.
constexpr int WSTR = 12;
__host__ __device__ constexpr int w_rows(int nkg) { return (2 * nkg + 3) & ~3; }

__device__ __forceinline__ float fmax_abs(float a, float b) { return fmaxf(a, fabsf(b)); }
// a value the compiler must keep in a register (it cannot rematerialize an asm result): used for
// per-task flags that register pressure would otherwise make it recompute at every use
__device__ __forceinline__ int opaque(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}
// ... only where registers allow it (otherwise the value itself: the builds at the register cap
// would spill the extra live registers)
template <bool ON>
__device__ __forceinline__ int keep(int v) { return ON ? opaque(v) : v; }

// shared-memory loads at a 32-bit shared-window address (no generic-address arithmetic)
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double2 lds_f64x2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}

// exact FP64 positions (both steps) of a body from its FP32 hi / lo rows (16-B aligned,
// (x0, x1, y0, y1[, z0, z1, 0, 0])): one vector load per row
template <int ND>
__device__ __forceinline__ void hilo_positions(const float* hp, const float* lp, double (&pj)[ND][2]) {
  const float4 h = *reinterpret_cast<const float4*>(hp), l = *reinterpret_cast<const float4*>(lp);
  pj[0][0] = (double)h.x + (double)l.x;
  pj[0][1] = (double)h.y + (double)l.y;
  pj[1][0] = (double)h.z + (double)l.z;
  pj[1][1] = (double)h.w + (double)l.w;
  if constexpr (ND == 3) {
    const float2 h2 = *reinterpret_cast<const float2*>(hp + 4), l2 = *reinterpret_cast<const float2*>(lp + 4);
    pj[ND - 1][0] = (double)h2.x + (double)l2.x;
    pj[ND - 1][1] = (double)h2.y + (double)l2.y;
  }
}

// append the sign bit of t (set = hit) below the bits already in m: (m << 1) | (t >> 31)
__device__ __forceinline__ unsigned push_hit(unsigned m, unsigned t) { return __funnelshift_l(t, m, 1); }

// 1/sqrt(q) in FP64 from the FP32 MUFU seed and one Newton step (relative error ~1e-14,  // @stage exact_math
// vs ~1e-16 for rsqrt(double); the seed needs q inside the FP32 normal range)
__device__ __forceinline__ double rsqrt_fast01(double q) {   // 1e-30 < q < 1
  float ys;   // (float)q is a normal number here: the flush-to-zero MUFU form needs no range fix-up
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(ys) : "f"((float)q));
  const double y = (double)ys;
  return y * fma(-0.5 * q, y * y, 1.5);
}

// Exact FP64 residual of one separation row (constraints.py:166-247, trig-free):
// r1 = delta * (1 - clip(rho, 1, d_max) / rho), coincident rows use alpha = 0, beta = pi/2.
// Returns false (r untouched) on the inactive range 1 <= rho <= d_max.
template <int ND>
__device__ __forceinline__ bool row_exact(const double (&d)[ND], double inv_a2, double inv_b2,
                                          double ax_a, double ax_b, double d_max,
                                          double coinc_sign, double (&r)[ND]) {
  double q = (d[0] * d[0] + d[1] * d[1]) * inv_a2;
  if (ND == 3) q = fma(d[ND - 1] * d[ND - 1], inv_b2, q);
  double f;
  if (q < 1.0 && q > 1e-30) {        // the active rows: 1 - 1/rho from the FP32 seed + Newton
    f = 1.0 - rsqrt_fast01(q);
  } else if (q < 1.0) {              // rho ~ 0: coincident rows, or an exact rsqrt
    if (q == 0.0) {
      r[0] = -ax_a * coinc_sign;
      r[1] = 0.0 * coinc_sign;
      if (ND == 3) r[ND - 1] = -ax_b * COS_HALF_PI * coinc_sign;
      return true;
    }
    f = 1.0 - rsqrt(q);
  } else if (q > d_max * d_max) {
    f = 1.0 - d_max * rsqrt(q);
  } else {
    return false;
  }
#pragma unroll
  for (int a = 0; a < ND; ++a) r[a] = f * d[a];
  return true;
}

// ---- DSMEM exchange primitives (sm_90+): stores into a peer CTA's shared memory that  // @stage cluster_prims
// complete a transaction count on the peer's mbarrier, so the receiver waits for its data
// instead of the whole cluster meeting at a barrier (which also costs a GPU-scope fence)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t dsmem_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT%=:\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t addr, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(addr), "d"(a), "d"(b), "r"(bar) : "memory");
}
// cluster exchange geometry: the G vector plus (S1, S2), padded to even length, in csize
// slices of SL (even) doubles; slice r has slice_len(r) live entries
__host__ __device__ inline int xch_tot(int nv) { return (nv + 3) & ~1; }
__host__ __device__ inline int xch_sl(int nv, int csize) { return ((xch_tot(nv) + csize - 1) / csize + 1) & ~1; }

#ifndef SFB_MINB
#define SFB_MINB 2
#endif

// Optional phase timing (build with -DSFB_PHASE_TIMING): thread 0 of every CTA accumulates
// clock64() deltas per phase into counters[b][4 + phase] (counters must then hold 12 slots).
#ifdef SFB_PHASE_TIMING
#define SFB_TMARK(ph)                                   \
  do {                                                  \
    if (tid == 0) {                                     \
      const long long now_ = clock64();                 \
      t_ph[ph] += now_ - t_last;                        \
      t_last = now_;                                    \
    }                                                   \
  } while (0)
#define SFB_TSUB(ph)                                    \
  do {                                                  \
    if (tid == 0) {                                     \
      const long long now_ = clock64();                 \
      t_ph[ph] += now_ - t_sub;                         \
      t_sub = now_;                                     \
    }                                                   \
  } while (0)
#else
#define SFB_TMARK(ph) do { } while (0)
#define SFB_TSUB(ph) do { } while (0)
#endif

// Race stress build (-DSFB_CHECKS, libsfb_checks.so, tools/race_stress.py): compute-sanitizer
// is closed on this GPU pool, so the concurrency protocols (the cluster's DSMEM / mbarrier
// exchange with parity-reused buffers, the split schedule's cross-CTA handoff, the
// per-warp task loop against the CTA barriers) are exercised by perturbation instead: at the
// points below a warp sleeps a pseudo-random 0..~4 us (seed KParams::jitter_seed), which
// reorders every race window; results must stay bitwise those of the plain build, and the
// device asserts below (trap on violation) check the protocol invariants.
#ifdef SFB_CHECKS
__device__ __forceinline__ void sfb_jitter(unsigned seed, unsigned site, unsigned it) {
  if (seed == 0u) return;
  unsigned h = seed * 0x9E3779B9u ^ (blockIdx.x * 0x85EBCA6Bu) ^ ((threadIdx.x >> 5) * 0xC2B2AE35u) ^
               (site * 0x27D4EB2Fu) ^ (it * 0x165667B1u);
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep((h >> 4) & 4095u);
}
#define SFB_JITTER(site, it) sfb_jitter(P.jitter_seed, (site), (unsigned)(it))
#define SFB_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define SFB_JITTER(site, it) do { } while (0)
#define SFB_CHECK(cond) do { } while (0)
#endif

#ifndef SFB_GREG
#define SFB_GREG 0   // n <= 32: axes of the G partials held in registers (the rest in per-lane smem slots)
#endif

// NJ: robot tile of one k-group (power of two >= n) for n <= 32; unused for n > 32 (BIG)
// BIG2 (n = 33..64, 2D): the n > 32 kernel capped at 128 registers, 8-warp CTAs, two per SM
// (16 warps per SM; the uncapped build needs 230 registers and runs 4-warp CTAs)
enum { PIECE_WHOLE = 0, PIECE_HEAD = 1, PIECE_TAIL = 2 };
// schedule slots in the misc words after the warp partials (sMisc[0..2] belong to the member solve)
enum { SCHED_MEMBER = 3, SCHED_PIECE = 4 };
// builds that run the split schedule: the 128-register n = 33..64 build and the 3D n <= 32
// builds have no register to spare for it (they would spill) and always run one member per CTA
template <int ND, bool BIG, bool BIG2>
__host__ __device__ constexpr bool split_build() { return ND == 2 && !BIG2; }
// One member's solve, evaluations it0 .. (max_iters or convergence), by one CTA (or one cluster).
// Split schedule (sf_solve_kernel): piece = PIECE_TAIL resumes the member from the state the
// previous CTA handed over (slot blockIdx.x - 1; xi / lambda in the member's outputs); for
// PIECE_HEAD the loop stops before evaluation `stop` (read from shared memory each iteration,
// so no register holds it across the solve) and hands the state to slot blockIdx.x.
// Returns true when the member finished (converged or reached max_iters), outputs written.
template <int ND, int NXI, int NJ, bool BIG, bool BIG2 = false, int MW = NW, bool TW = false>
__device__ __forceinline__ bool sf_member(const KParams& P, const int it0, const int piece,
                                          const int stop) {  // @stage setup
  constexpr int ND2 = (ND == 2) ? 4 : 8;   // floats per body per k-group
  constexpr int NXP = nxi_pad(NXI);        // padded coefficient stride in shared memory
  constexpr bool KEEP = !BIG && ND == 2;   // per-task flags pinned in registers (see keep())
  constexpr int OS = (ND == 2) ? 4 : 8;    // floats per static obstacle
  constexpr unsigned FULL = 0xffffffffu;
  extern __shared__ __align__(16) unsigned char smem[];
  // split builds: the member's index lives in shared memory (the schedule slot the kernel
  // writes before the solve) and is re-read where used, so the compiler need not keep it live
  auto member = [&]() -> int {
    if constexpr (!split_build<ND, BIG, BIG2>()) return blockIdx.x / P.csize;
    return (int)*reinterpret_cast<const unsigned*>(smem + P.L.red + NW_RED * 4 * 8 + SCHED_MEMBER * 4);
  };

  // a member is owned by a cluster of csize CTAs; CTA rank crank owns a contiguous slice
  // of the k-group tasks and all ranks run the (identical) KKT step redundantly
  const int csize = P.csize;
  const int crank = csize > 1 ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nw = BIG ? P.nw : NW, nt = nw * 32;   // n <= 32 always runs NW warps (compile-time strides)
  static_assert(MW == NW || BIG2, "only the capped n > 32 build comes in a 16-warp variant");
  const int n = P.n, m = P.m, MP = P.MP, K1 = P.K1, NB = P.NB, NKG = P.NKG;
  const int nv = ND * n * NXI;       // dense outputs per member
  const int nrows = ND * n;          // (axis, robot) rows
  const int inst = P.member_instance[member()];

  double* sXi = reinterpret_cast<double*>(smem + P.L.xi);    // [ND*n][NXP]
  double* sLam = reinterpret_cast<double*>(smem + P.L.lam);  // [ND*n][NXP]
  double* sTgt = reinterpret_cast<double*>(smem + P.L.tgt);  // [ND*n][NXI] (projection target)
  double* sW = reinterpret_cast<double*>(smem + P.L.w);      // [w_rows(NKG)][WSTR], zero padded
  double* sE = reinterpret_cast<double*>(smem + P.L.e);      // [NB][NXI]
  double* sQ = reinterpret_cast<double*>(smem + P.L.q);      // [NXI][NXI]
  double* sPxx = reinterpret_cast<double*>(smem + P.L.pxx);
  double* sPxb = reinterpret_cast<double*>(smem + P.L.pxb);
  double* sPB = reinterpret_cast<double*>(smem + P.L.pb);
  double* sDxx = reinterpret_cast<double*>(smem + P.L.dxx);
  double* sDxb = reinterpret_cast<double*>(smem + P.L.dxb);
  double* sG = reinterpret_cast<double*>(smem + P.L.g);      // [ND*n][NXI]
  // boundary values b [ND*n][NB] stay in global memory (read once per iteration, L1-resident)
  const double* __restrict__ gBv = P.bvals + (size_t)inst * ND * n * NB;
  double* sRed = reinterpret_cast<double*>(smem + P.L.red);  // [NW][4] + misc
  double* sObsAx = reinterpret_cast<double*>(smem + P.L.obs_ax);   // [MP][4] inv_a2 inv_b2 a b
  float* sObsThr = reinterpret_cast<float*>(smem + P.L.obs_thr);   // [2][MP] thr, kappa
  double* sObsC = reinterpret_cast<double*>(smem + P.L.obs_c);     // [MP][ND] exact centers (static)
  float* sObsS = reinterpret_cast<float*>(smem + P.L.obs_s);       // [MP][OS] static: -x -y (-z) -thr (kappa)
  float* sObs = reinterpret_cast<float*>(smem + P.L.obs);          // [NKG][MP][ND2] (dynamic)
  float* sPmax = reinterpret_cast<float*>(smem + P.L.pmax);        // [kgs][8] (n > 32)
  unsigned char* uni = smem + keep<BIG>(P.L.uni);
  const int NROW = BIG ? n : NJ;                                    // bodies per k-group row
  // n > 32: positions of every k-group are shared by the robot-block warps of that k-group;
  // n <= 32: a warp holds all robots of its k-groups, so it owns a private position row
  float* sPos = reinterpret_cast<float*>(uni);                      // BIG [NKG][NROW][ND2] / [nw][32/NJ][NJ][ND2]
  float* sLo = sPos + (size_t)P.kgs * NROW * ND2;                   // [kgs][NROW][ND2] lo (BIG)
  // n > 32: a k-group's positions live in ring slot 2 wk + (task parity) of its worker: the
  // worker's named barrier at the next task orders all reads of a slot before its reuse
  double* sSlot = reinterpret_cast<double*>(uni);                   // G partial slots (BIG)
  // n <= 32: per-lane G partials [nw][NXI][ND][32] (conflict-free, lane-contiguous)
  double* sGl = reinterpret_cast<double*>(smem + P.L.gl);
  // TBL (one k-group row of 32 robots per warp task): g_i(k) goes to a [k][axis * n + i] table
  // (row stride TS, XOR-swizzled columns: conflict-free DMMA fragment loads) for the
  // tensor-core contraction, instead of per-lane partials of G
  constexpr bool TBL = !BIG;   // (n <= 16: 32 / NJ k-groups per warp task)
  // TW (the 16-warp n = 33..64 build when its table fits): the same table-based positions
  // (phase A) and DMMA contraction as TBL, with robot blocks of 32 as tasks
  static_assert(!TW || (BIG && BIG2 && MW == 16 && ND == 2), "table build: 16-warp n = 33..64, 2D");
  constexpr bool TAB = TBL || TW;
  constexpr int CA = TW ? 64 : (NJ < 16 ? 16 : NJ);   // table columns per axis (>= 16: the swizzle stays in range)
  double* sTab = sGl;
  // column of (axis a, robot i) in the g table: a * CA + i (CA columns per axis whatever n is, so
  // the axis is an immediate offset and the swizzle only touches the robot index)
  const int TS = tab_stride(ND * CA);
  // KKT scratch (aliases the union region (BIG) / the per-lane partials or g table after the
  // reduction; TBL rows it overwrites are rewritten by their task, or masked, before use)
  double* sD = reinterpret_cast<double*>(BIG ? uni : smem + P.L.gl);  // [ND*n][NXI]
  // TBL: the boundary rows u = b - E xi get their own buffer (the KKT scratch aliases the g
  // table, which the task loop is still writing when the lighter warps compute u)
  double* sU = TBL ? reinterpret_cast<double*>(smem + P.L.ub) : sD + nv;   // [ND*n][NB]
  double* sSD = sD + nv + ND * n * NB;                              // [ND][NXI] (KKT scratch)
  double* sSU = TBL ? sU + ND * n * NB : sSD + ND * NXI;             // [ND][NB]

  const ConstOff co = ConstOff::make(K1, NXI, NB);
  // (axis, robot) row of a dense index o = ai * NXI + c without runtime division
  auto split = [&](int o, int& ai, int& c, int& a, int& ii) {
    ai = o / NXI;
    c = o - ai * NXI;
    a = (ai >= n) + (ND == 3 && ai >= 2 * n);
    ii = ai - a * n;
  };

  // ------------------------------------------------------------------ setup
#ifdef SFB_CHECKS
  {
    unsigned dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    SFB_CHECK((unsigned)P.L.total <= dyn && (unsigned)P.L.uni + (unsigned)P.L.uni_bytes <= dyn);
    SFB_CHECK(P.csize == 1 || (unsigned)P.L.xg + (unsigned)(P.csize * xch_sl(ND * P.n * NXI, P.csize) * 8 + 16) <= dyn);
  }
#endif
  for (int idx = tid; idx < w_rows(NKG) * WSTR; idx += nt) {
    const int k = idx / WSTR, c = idx - k * WSTR;
    sW[idx] = (k < K1 && c < NXI) ? P.consts[co.W + k * NXI + c] : 0.0;
  }
  if (TAB) {   // g-table rows K1 .. (K1 rounded up to 4) are read by the contraction, never written
    for (int idx = tid; idx < (((K1 + 3) & ~3) - K1) * TS; idx += nt) sTab[(size_t)K1 * TS + idx] = 0.0;
  }
  for (int idx = tid; idx < NB * NXI; idx += nt) sE[idx] = P.consts[co.E + idx];
  for (int idx = tid; idx < NXI * NXI; idx += nt) {
    sQ[idx] = P.consts[co.Q + idx];
    sPxx[idx] = P.consts[co.Pxx + idx];
    sDxx[idx] = P.consts[co.Dxx + idx];
  }
  for (int idx = tid; idx < NXI * NB; idx += nt) {
    sPxb[idx] = P.consts[co.Pxb + idx];
    sDxb[idx] = P.consts[co.Dxb + idx];
  }
  if (TBL) {   // E2's B operand, fragment-ordered and zero padded: one unconditional LDS.64 each
    const int KT = NXI + NB, nks = (KT + 3) >> 2;
    for (int idx = tid; idx < nks * 64; idx += nt) {
      const int ks = idx >> 6, c = ((idx >> 5) & 1) * 8 + ((idx & 31) >> 2), k = 4 * ks + (idx & 3);
      sPB[idx] = (c < NXI && k < KT) ? ((k < NXI) ? P.consts[co.Pxx + c * NXI + k]
                                                  : P.consts[co.Pxb + c * NB + (k - NXI)]) : 0.0;
    }
  }
  {
    // a handed-over member resumes from the iterate its previous CTA left in the outputs
    // (written by another SM in this launch: read through L2)
    const bool resume = piece == PIECE_TAIL;
    const double* x0 = (resume ? P.xi : P.xi0) + (size_t)member() * nv;
    const double* l0 = (resume ? P.lam : P.lam0) + (size_t)member() * nv;
    const double* t0 = P.target ? P.target + (size_t)member() * nv : nullptr;
    for (int o = tid; o < nv; o += nt) {
      const int ai = o / NXI, c = o - ai * NXI;
      sXi[ai * NXP + c] = resume ? __ldcg(x0 + o) : x0[o];
      sLam[ai * NXP + c] = resume ? __ldcg(l0 + o) : l0[o];
      sTgt[o] = t0 ? t0[o] : 0.0;
    }
  }
  // xi's padding columns feed the positions' DMMA (times a zero W column): keep them zero
  for (int idx = tid; idx < ND * n * (NXP - NXI); idx += nt) {
    const int r = idx / (NXP - NXI);
    sXi[r * NXP + NXI + (idx - r * (NXP - NXI))] = 0.0;
  }
  // obstacles, padded to MP (multiple of 4) with far-away dummies that never screen in
  for (int o = tid; o < MP; o += nt) {
    float* st = sObsS + o * OS;
    if (o < m) {
      const double* oa = P.obs_axes + ((size_t)inst * m + o) * 3;
      const double a = oa[0], bb = oa[2];
      sObsAx[o * 4 + 0] = 1.0 / (a * a);
      sObsAx[o * 4 + 1] = 1.0 / (bb * bb);
      sObsAx[o * 4 + 2] = a;
      sObsAx[o * 4 + 3] = bb;
      const float thr = (float)(a * a * (1.0 + 2e-3)), kap = (float)((a * a) / (bb * bb));
      sObsThr[o] = thr;
      sObsThr[MP + o] = kap;
#pragma unroll
      for (int a2 = 0; a2 < ND; ++a2) {
        const double c0 = P.obs_pos[(((size_t)inst * ND + a2) * m + o) * K1];
        sObsC[o * ND + a2] = c0;
        st[a2] = -(float)c0;
      }
      st[ND] = -thr;
      if (ND == 3) { st[4] = kap; st[5] = st[6] = st[7] = 0.f; } else { st[3] = 0.f; }
    } else {
      sObsThr[o] = 0.f;
      sObsThr[MP + o] = 0.f;
#pragma unroll
      for (int a2 = 0; a2 < OS; ++a2) st[a2] = 0.f;
      st[0] = -PAD_SMEM;                     // dummy at +3e30: never within any threshold
    }
  }
  float obs_absmax = 0.f, obs_axmin = INFINITY;
  for (int o = tid; o < m; o += nt) {
    const double* oa = P.obs_axes + ((size_t)inst * m + o) * 3;
    obs_axmin = fminf(obs_axmin, (float)(ND == 3 ? fmin(oa[0], oa[2]) : oa[0]));
  }
  const int NKGO = P.obs_static ? 0 : NKG;
  for (int idx = tid; idx < NKGO * MP; idx += nt) {
    const int kg = idx / MP, o = idx - kg * MP;
    float* dst = sObs + (size_t)idx * ND2;
#pragma unroll
    for (int a = 0; a < ND; ++a) {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int k = 2 * kg + kk;
        float v = PAD_SMEM;
        if (o < m && k < K1) v = (float)P.obs_pos[(((size_t)inst * ND + a) * m + o) * K1 + k];
        dst[a * 2 + kk] = v;
      }
    }
    if (ND == 3) dst[6] = dst[7] = 0.f;
  }
  for (int idx = tid; idx < m * K1; idx += nt) {
    const int o = idx / K1, k = idx - o * K1;
#pragma unroll
    for (int a = 0; a < ND; ++a)
      obs_absmax = fmax_abs(obs_absmax, (float)P.obs_pos[(((size_t)inst * ND + a) * m + o) * K1 + k]);
  }
  unsigned* sMisc = reinterpret_cast<unsigned*>(sRed + NW_RED * 4);
  if (tid == 0) {
    sMisc[0] = 0u;
    sMisc[1] = __float_as_uint(INFINITY);
    sMisc[2] = piece == PIECE_HEAD ? (unsigned)stop : 0xffffffffu;   // split schedule stop
  }
  __syncthreads();
  if (obs_absmax > 0.f) atomicMax(&sMisc[0], __float_as_uint(obs_absmax));
  if (obs_axmin < INFINITY) atomicMin(&sMisc[1], __float_as_uint(obs_axmin));
  __syncthreads();
  obs_absmax = __uint_as_float(sMisc[0]);
  // compact mode (n <= 32, at most 32 static obstacles; for n > 32 the per-lane candidate loop
  // measured slower than the broadcast screen): obstacle rows are nominated by a grid over the
  // obstacles' (x, y) contact discs instead of an FP32 test of every obstacle. A cell lists
  // obstacle o if its rectangle, widened by 1e-3 of a cell, meets the disc of radius
  // 1.001 a_o + 1e-6 around the centre: every row the FP32 screen could flag (|p - c| < a
  // sqrt(1 + 2e-3) with FP32 positions) lies in such a cell, and in 3D rho >= |(dx, dy)| / a,
  // so no active row is lost; candidates are then confirmed by the screen's own FP32 test.
  const bool compact = keep<KEEP>(P.compact && (m == 0 || P.obs_static) ? 1 : 0) != 0;
  unsigned* sGrid = reinterpret_cast<unsigned*>(smem + P.L.grid);
  double* sKD = reinterpret_cast<double*>(smem + P.L.kc);
  float* sKF = reinterpret_cast<float*>(sKD + KC_NDBL);
  if (compact && m > 0) {
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (int o = 0; o < m; ++o) {
      const double rg = sObsAx[o * 4 + 2] * 1.001 + 1e-6;
      x0 = fmin(x0, sObsC[o * ND] - rg);
      x1 = fmax(x1, sObsC[o * ND] + rg);
      y0 = fmin(y0, sObsC[o * ND + 1] - rg);
      y1 = fmax(y1, sObsC[o * ND + 1] + rg);
    }
    const double hx = (x1 - x0) / GRID, hy = (y1 - y0) / GRID;
    if (tid == 0) {
      // cell coordinate u = (x - x0) / hx as one FMA: x * (1 / hx) + (-x0 / hx)
      sKF[KC_F_GX0] = (float)(-x0 / hx);
      sKF[KC_F_GY0] = (float)(-y0 / hy);
      sKF[KC_F_GIX] = (float)(1.0 / hx);
      sKF[KC_F_GIY] = (float)(1.0 / hy);
    }
    for (int cidx = tid; cidx < GRID * GRID; cidx += nt) {
      const int cy = cidx / GRID, cx = cidx - cy * GRID;
      const double rx0 = x0 + cx * hx - 1e-3 * hx, rx1 = x0 + (cx + 1) * hx + 1e-3 * hx;
      const double ry0 = y0 + cy * hy - 1e-3 * hy, ry1 = y0 + (cy + 1) * hy + 1e-3 * hy;
      unsigned bits = 0u;
      for (int o = 0; o < m; ++o) {
        const double ox = sObsC[o * ND], oy = sObsC[o * ND + 1];
        const double dx = fmin(fmax(ox, rx0), rx1) - ox, dy = fmin(fmax(oy, ry0), ry1) - oy;
        const double rg = sObsAx[o * 4 + 2] * 1.001 + 1e-6;
        if (dx * dx + dy * dy <= rg * rg) bits |= 1u << o;
      }
      sGrid[cidx] = bits;
    }
    __syncthreads();
  }
  // cluster exchange: receive buffer [csize][SL] then two mbarriers (reduce-scatter, all-gather)
  const int xtot = xch_tot(nv), xSL = xch_sl(nv, csize);
  double* xrecv = reinterpret_cast<double*>(smem + P.L.xg);
  const uint32_t xbar1 = smem_u32(xrecv + (size_t)csize * xSL), xbar2 = xbar1 + 8;
  if (csize > 1) {
    if (tid == 0) {
      mbar_init(xbar1, 1);
      mbar_init(xbar2, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cooperative_groups::this_cluster().sync();   // peers started and their barriers exist
  }

  const double ra0 = P.pair_axes[(size_t)inst * 3 + 0], rb0 = P.pair_axes[(size_t)inst * 3 + 2];
  if (tid == 0) {
#pragma unroll
    for (int a = 0; a < ND; ++a) {
      const double lo = P.box[((size_t)inst * 2 + 0) * ND + a], hi = P.box[((size_t)inst * 2 + 1) * ND + a];
      sKD[KC_BLO + a] = lo;
      sKD[KC_BHI + a] = hi;
      const float bmg = 1e-4f * (1.f + (float)fmax(fabs(lo), fabs(hi)));
      sKF[KC_F_BLO + a] = (float)lo + bmg;
      sKF[KC_F_BHI + a] = (float)hi - bmg;
    }
    sKD[KC_INV_A2] = 1.0 / (ra0 * ra0);
    sKD[KC_INV_B2] = 1.0 / (rb0 * rb0);
    sKD[KC_RA] = ra0;
    sKD[KC_RB] = rb0;
    sKD[KC_DMAX] = P.d_max;
  }
  __syncthreads();
  const float r_thr = (float)(ra0 * ra0 * (1.0 + 2e-3));
  const float r_kap = (float)((ra0 * ra0) / (rb0 * rb0));
  // FP32 positions carry ~2^-24 |p| error: the screen margin (1e-3 of the contact
  // distance) covers it while every |p| <= plim; beyond, rows go exact
  // ... and rows beyond the clip (rho > d_max, constraints.py:199-201) are active too: with c the
  // largest |coordinate| of positions and obstacle centres, every row has rho <= 2 sqrt(n_d) c /
  // a_min, so below c = d_max a_min / (2 sqrt(n_d)) none is; above, every row goes exact
  const float amin_all = fminf(__uint_as_float(sMisc[1]), (float)(ND == 3 ? fmin(ra0, rb0) : ra0));
  const float plim = fminf(P.plim * amin_all,
                           (float)(P.d_max * (1.0 - 1e-4) / (2.0 * sqrt((double)ND))) * amin_all);
  const double* opos = P.obs_pos + (size_t)inst * ND * m * K1;
  // static obstacles in one chunk: the exact pair and obstacle rows run in one loop
  const bool merge_rows = keep<KEEP || BIG>(P.obs_static && m > 0 && MP <= 32 ? 1 : 0) != 0;

  // lane -> (robot, k-group) mapping
  constexpr int LW = BIG ? 32 : NJ, SUB = 32 / LW;
  int sub, rbk, wk, nwk;
  if (BIG) {
    sub = 0;
    rbk = warp & (P.RB - 1); wk = warp / P.RB; nwk = nw / P.RB;
  } else {
    sub = lane / LW;
    rbk = 0; wk = warp; nwk = nw;
  }
  const int i = BIG ? keep<BIG>(rbk * 32 + lane) : lane % LW;
  const bool robot_ok = keep<KEEP || BIG>(i < n ? 1 : 0) != 0;
  const int ic = keep<KEEP>(robot_ok ? i : n - 1);
  const int NTS = (NKG + SUB - 1) / SUB;
  const int ts_lo = (NTS * crank) / csize, ts_hi = (NTS * (crank + 1)) / csize;
  const double* xrow = sXi + (size_t)ic * NXP;   // axis a at + a * n * NXP

#ifdef SFB_PHASE_TIMING
  long long t_ph[18] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
  long long t_last = clock64(), t_sub = t_last;
#endif
  double last_fp = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  double eq_max = 0.0, eql = 0.0;
  double fpp = 0.0;   // per-lane ||dlambda||^2 + ||dxi||^2 partial of the last KKT step
  if (piece == PIECE_TAIL) {   // the per-thread carries of the previous CTA (same thread, same values)
    const double* hb = P.hand + (size_t)(blockIdx.x - 1) * 2 * nt;
    fpp = __ldcg(hb + tid);
    eql = __ldcg(hb + nt + tid);
  }
  bool finished = true;
  // per-thread counts fit 32 bits (rows of one lane over one solve); summed in 64 bits at the end
  unsigned c_exact = 0, c_active = 0, c_screen = 0, c_evals = 0;

  for (int it = it0;; ++it) {  // @stage iter_top
    if (split_build<ND, BIG, BIG2>() && it == (int)sMisc[2]) {
      // split schedule: hand the state before evaluation it to the next CTA (xi / lambda
      // through the member's outputs, the per-thread carries through the handoff slot)
      double* xo = P.xi + (size_t)member() * nv;
      double* lo = P.lam + (size_t)member() * nv;
      for (int o = tid; o < nv; o += nt) {
        const int ai = o / NXI, c = o - ai * NXI;
        xo[o] = sXi[ai * NXP + c];
        lo[o] = sLam[ai * NXP + c];
      }
      double* hb = P.hand + (size_t)blockIdx.x * 2 * nt;
      hb[tid] = fpp;
      hb[nt + tid] = eql;
      finished = false;
      break;
    }
    // -------------------------------------------- A (TBL): positions of every step on DMMA  // @stage A_positions
    // P (k x col) = W (k x c) . X^T (c x col), X[col][c] = xi of the (axis, robot) row col, into
    // the g table (sTab[k][col ^ tab_swz(k)]): warp per 8 x 8 tile, k-dim c in steps of 4. A
    // task reads its own and its partners' positions from there and overwrites its rows with
    // g_i(k) once its rows are done (no other task reads them). Rows outside this CTA's steps
    // [klo, khi) are not stored (the contraction masks them).
    if (TAB) {
      const int ncol = ND * CA, ntn = ncol >> 3;         // table columns a * CA + i
      const int klo = 2 * SUB * ts_lo, khi = min(K1, 2 * SUB * ts_hi);
      const int mt0 = klo >> 3, ntm = ((khi + 7) >> 3) - mt0;
      const int rq = lane >> 2, kq = lane & 3;
      constexpr int NKS = (NXI + 3) / 4;
      // A warp owns a column tile (its B fragments loaded once) and every G-th row tile of
      // it (G row groups per column tile so that every warp has work). No operand masks: W is
      // zero for c >= NXI and xi's padding columns are zero (set up once, never written), or
      // (NXP < 4 NKS) the next row's finite value times that zero; rows past K1 and columns
      // past ND n read finite neighbouring buffers and are never stored.
      const int G = (nw + ntn - 1) / ntn;
      const int swl = (rq & 3) << 2;                 // tab_swz of every row this lane stores
      for (int item = warp; item < ntn * G; item += nw) {
        const int rg = item / ntn, nt2 = item - rg * ntn;
        const int colb = nt2 * 8 + rq, col = nt2 * 8 + 2 * kq;
        // table column a * CA + i <- xi row a * n + i (columns of robots i >= n: robot 0's values,
        // never read by a task, and the contraction does not store them)
        const int xrow_b = (colb / CA) * n + ((colb & (CA - 1)) < n ? (colb & (CA - 1)) : 0);
        double bfr[NKS];
#pragma unroll
        for (int ks = 0; ks < NKS; ++ks) {
          const int c = 4 * ks + kq;
          bfr[ks] = (4 * NKS > NXP && c >= NXI) ? 0.0 : sXi[xrow_b * NXP + c];   // crossed into the next row
        }
        const bool pair_ok = col + 1 < ncol, one_ok = col < ncol;
        const double* wa = sW + ((mt0 + rg) * 8 + rq) * WSTR + kq;
        double* dst = sTab + ((mt0 + rg) * 8 + rq) * TS + (col ^ swl);
        int kr = (mt0 + rg) * 8 + rq;
        for (int mt = rg; mt < ntm; mt += G, wa += 8 * G * WSTR, dst += 8 * G * TS, kr += 8 * G) {
          double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
          for (int ks = 0; ks < NKS; ++ks)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc0), "+d"(acc1) : "d"(wa[4 * ks]), "d"(bfr[ks]));
          if (kr >= klo && kr < khi) {
            if (pair_ok) *reinterpret_cast<double2*>(dst) = make_double2(acc0, acc1);
            else if (one_ok) *dst = acc0;
          }
        }
      }
      __syncthreads();
    }
    // -------------------------------------------- A/B/C per k-group task
    // G partials (not TBL): the first RA axes in registers, the rest in per-lane smem slots
    constexpr int RA = BIG ? ND : (SFB_GREG > ND ? ND : SFB_GREG);
    double Gp[RA > 0 ? RA : 1][NXI];
    double* gl = sGl + (size_t)warp * NXI * ND * 32 + lane;          // this lane's partials, stride 32
    if (!TAB) {
#pragma unroll
      for (int a = 0; a < ND; ++a)
#pragma unroll
        for (int c = 0; c < NXI; ++c) {
          if (a < RA) Gp[a < RA ? a : 0][c] = 0.0;
          else gl[(c * ND + a) * 32] = 0.0;
        }
    }
    float* posw = sPos + (size_t)(warp * SUB + sub) * NJ * ND2;        // !BIG: this k-group's row
    double s1 = 0.0, s2 = 0.0;

    SFB_JITTER(1, it);
    for (int ts = ts_lo + wk, tcnt = 0; ts < ts_hi; ts += nwk, ++tcnt) {
      SFB_JITTER(2, it * 64 + ts);
      const int pslot = BIG ? 2 * wk + (tcnt & 1) : 0;
      const int kg_raw = ts * SUB + sub;
      const bool kg_ok = SUB == 1 || kg_raw < NKG;   // one k-group per task: ts < NTS = NKG
      const int kg = kg_ok ? kg_raw : NKG - 1;
      const bool live = robot_ok && kg_ok;
      const bool has1 = keep<KEEP || BIG>(2 * kg + 1 < K1 ? 1 : 0) != 0;
      const double* w0r = sW + (size_t)(2 * kg) * WSTR;   // W rows of the two steps
      const double* w1r = w0r + WSTR;
#ifdef SFB_PHASE_TIMING
      if (tid == 0) t_sub = clock64();
#endif

      // A: exact positions of the lane's robot at the two steps  // @stage A_positions
      // (TBL: from the table phase A filled; a missing second step or an idle lane reads a
      // valid cell of the task's first step)
      const int k0 = 2 * kg, k1 = has1 ? k0 + 1 : k0;
      const double* tr0 = sTab + (size_t)k0 * TS;
      const double* tr1 = sTab + (size_t)k1 * TS;
      const int sw0 = tab_swz(k0), sw1 = tab_swz(k1);
      double p[ND][2];
#pragma unroll
      for (int a = 0; a < ND; ++a) {
        if (TAB) {
          p[a][0] = tr0[a * CA + (ic ^ sw0)];
          p[a][1] = tr1[a * CA + (ic ^ sw1)];
        } else {
          p[a][0] = p[a][1] = 0.0;
        }
      }
#pragma unroll
      for (int c = 0; !TAB && c + 1 < NXI; c += 2) {
        const double2 u0 = *reinterpret_cast<const double2*>(w0r + c);
        const double2 u1 = *reinterpret_cast<const double2*>(w1r + c);
#pragma unroll
        for (int a = 0; a < ND; ++a) {
          const double2 x = *reinterpret_cast<const double2*>(xrow + a * n * NXP + c);
          p[a][0] = fma(u0.y, x.y, fma(u0.x, x.x, p[a][0]));
          p[a][1] = fma(u1.y, x.y, fma(u1.x, x.x, p[a][1]));
        }
      }
      if (!TAB && (NXI & 1)) {
        const double u0 = w0r[NXI - 1], u1 = w1r[NXI - 1];
#pragma unroll
        for (int a = 0; a < ND; ++a) {
          const double x = xrow[a * n * NXP + NXI - 1];
          p[a][0] = fma(u0, x, p[a][0]);
          p[a][1] = fma(u1, x, p[a][1]);
        }
      }
      float own[ND][2];
      float pabs = 0.f;
      {
        float hv[ND2];
#pragma unroll
        for (int a = 0; a < ND; ++a) {
          const float h0 = (float)p[a][0];
          const float h1 = (float)p[a][1];
          pabs = fmaxf(pabs, fmaxf(fabsf(h0), fabsf(h1)));
          hv[2 * a] = robot_ok ? h0 : PAD_SMEM;
          hv[2 * a + 1] = (robot_ok && has1) ? h1 : PAD_SMEM;
          own[a][0] = live ? h0 : PAD_OWN;
          own[a][1] = (live && has1) ? h1 : PAD_OWN;
        }
        if (ND == 3) hv[6] = hv[7] = 0.f;
        if (BIG ? (kg_ok && robot_ok) : true) {
          float4* dst = reinterpret_cast<float4*>(BIG ? sPos + ((size_t)pslot * NROW + i) * ND2 : posw + i * ND2);
          dst[0] = make_float4(hv[0], hv[1], hv[2], hv[3]);
          if (ND == 3) dst[1] = make_float4(hv[4], hv[5], hv[6], hv[7]);
          if (BIG && !TW) {   // (TW: exact partner positions come from the table)
            float lv[ND2];
#pragma unroll
            for (int a = 0; a < ND; ++a) {
              lv[2 * a] = (float)(p[a][0] - (double)hv[2 * a]);
              lv[2 * a + 1] = has1 ? (float)(p[a][1] - (double)hv[2 * a + 1]) : 0.f;
            }
            if (ND == 3) lv[6] = lv[7] = 0.f;
            float4* dl = reinterpret_cast<float4*>(sLo + ((size_t)pslot * NROW + i) * ND2);
            dl[0] = make_float4(lv[0], lv[1], lv[2], lv[3]);
            if (ND == 3) dl[1] = make_float4(lv[4], lv[5], lv[6], lv[7]);
          }
        }
      }
      pabs = __uint_as_float(__reduce_max_sync(FULL, __float_as_uint(pabs)));
      if (BIG) {
        if (lane == 0) sPmax[pslot * 8 + rbk] = pabs;
        // every robot block of this k-group must have stored its positions
        asm volatile("bar.sync %0, %1;" ::"r"(1 + wk), "r"(P.RB * 32) : "memory");
        for (int r = 0; r < P.RB; ++r) pabs = fmaxf(pabs, sPmax[pslot * 8 + r]);
      } else {
        __syncwarp();
      }
      // conservative FP32 screening is valid while positions stay below plim
      const bool force = !(fmaxf(pabs, obs_absmax) <= plim);
      const float2 nx = make_float2(-own[0][0], -own[0][1]);
      const float2 ny = make_float2(-own[1][0], -own[1][1]);
      const float2 nz = (ND == 3) ? make_float2(-own[ND - 1][0], -own[ND - 1][1]) : make_float2(0.f, 0.f);
      const int nsteps = live ? (has1 ? 2 : 1) : 0;
      // obstacle-grid candidates of the lane's two positions, looked up before the pair screen
      // so the shared-memory latency overlaps it (the FMA's rounding moves a cell coordinate by
      // ~1e-5 of a cell, well inside the cells' 1e-3 widening)
      // (n <= 32 only: the n > 32 builds have no register to keep it across the pair chunks)
      auto grid_lookup = [&]() -> unsigned {
        if (!live) return 0u;
        const float4 gk = *reinterpret_cast<const float4*>(sKF + KC_F_GX0);   // bx by ax ay
        const float2 ux = __ffma2_rn(make_float2(own[0][0], own[0][1]), make_float2(gk.z, gk.z), make_float2(gk.x, gk.x));
        const float2 uy = __ffma2_rn(make_float2(own[1][0], own[1][1]), make_float2(gk.w, gk.w), make_float2(gk.y, gk.y));
        auto cell = [&](float u, float v) -> unsigned {
          const int cx = __float2int_rd(u), cy = __float2int_rd(v);
          return ((unsigned)(cx | cy) < (unsigned)GRID) ? sGrid[cy * GRID + cx] : 0u;
        };
        unsigned c = cell(ux.x, uy.x);
        if (has1) c |= cell(ux.y, uy.y);
        return c;
      };
      const unsigned grid_cand = (TBL && compact && !force) ? grid_lookup() : 0u;
      SFB_TSUB(6);

      double g[ND][2];  // @stage B_pair_screen
#pragma unroll
      for (int a = 0; a < ND; ++a) g[a][0] = g[a][1] = 0.0;

      // pair screen of one chunk of 32 bodies: bit j set if body j0 + j may be within contact
      auto pair_screen = [&](int j0, int jc) -> unsigned {
        const float2 thr2 = make_float2(-r_thr, -r_thr);
        const float* base = BIG ? sPos + ((size_t)pslot * NROW + j0) * ND2 : posw;
        unsigned mm = 0u;
        auto screen = [&](const float* bp, unsigned& mm) {
          const float4 v = *reinterpret_cast<const float4*>(bp);
          const float2 dx = __fadd2_rn(make_float2(v.x, v.y), nx);
          const float2 dy = __fadd2_rn(make_float2(v.z, v.w), ny);
          float2 q = __ffma2_rn(dy, dy, thr2);
          q = __ffma2_rn(dx, dx, q);
          if (ND == 3) {
            const float4 v2 = *reinterpret_cast<const float4*>(bp + 4);
            const float2 dz = __fadd2_rn(make_float2(v2.x, v2.y), nz);
            q = __ffma2_rn(__fmul2_rn(dz, make_float2(r_kap, r_kap)), dz, q);
          }
          mm = push_hit(mm, __float_as_uint(q.x) | __float_as_uint(q.y));
        };
        if constexpr (BIG) {
          if (jc == 32) {   // full chunk: unrolled, partner rows at immediate offsets
#pragma unroll
            for (int j = 0; j < 32; ++j) screen(base + j * ND2, mm);
            return __brev(mm);
          }
#pragma unroll 4
          for (int j = 0; j < jc; ++j) screen(base + (size_t)j * ND2, mm);
          return __brev(mm) >> (32 - jc);
        } else {
#pragma unroll
          for (int j = 0; j < NJ; ++j) screen(base + j * ND2, mm);
          return (__brev(mm) >> (32 - NJ)) & ((jc >= 32) ? FULL : ((1u << jc) - 1u));
        }
      };

      // obstacle screen of the chunk o0 .. o0 + 31: bit o set if obstacle o0 + o may be within
      // contact at one of the lane's steps (always 0 past MP or for an idle lane)
      auto obs_screen = [&](const int o0) -> unsigned {  // @stage B_obs_screen
        if (o0 >= MP) return 0u;
        const int oc = min(32, MP - o0);
        unsigned mask = 0u;
        if (!force) {
          unsigned mm = 0u;
          if (compact) {
            // grid candidates of the lane's two positions, each confirmed by the FP32 test
            // (per lane: a robot is near few obstacles)
            // (cells looked up before the pair screen: grid_cand)
            unsigned cand = o0 != 0 ? 0u : (TBL ? grid_cand : grid_lookup());
            while (cand) {
              const int o = __ffs(cand) - 1;
              cand &= cand - 1u;
              const float4 v = *reinterpret_cast<const float4*>(sObsS + o * OS);
              const float2 dx = __fadd2_rn(make_float2(v.x, v.x), make_float2(own[0][0], own[0][1]));
              const float2 dy = __fadd2_rn(make_float2(v.y, v.y), make_float2(own[1][0], own[1][1]));
              float2 q;
              if (ND == 3) {
                const float4 v2 = *reinterpret_cast<const float4*>(sObsS + o * OS + 4);
                const float2 dz = __fadd2_rn(make_float2(v.z, v.z),
                                             make_float2(own[ND - 1][0], own[ND - 1][1]));
                q = __ffma2_rn(__fmul2_rn(dz, make_float2(v2.x, v2.x)), dz, make_float2(v.w, v.w));
                q = __ffma2_rn(dy, dy, q);
              } else {
                q = __ffma2_rn(dy, dy, make_float2(v.z, v.z));
              }
              q = __ffma2_rn(dx, dx, q);
              if ((int)(__float_as_uint(q.x) | __float_as_uint(q.y)) < 0) mm |= 1u << o;
            }
            return live ? mm : 0u;   // bit o = obstacle o (one chunk: MP <= 32)
          } else if (P.obs_static) {
            // one row per obstacle: (-x, -y[, -z], -thr[, kappa]); packed ops broadcast the scalars
            const float* ob = sObsS + (size_t)o0 * OS;
            for (int o4 = 0; o4 < oc; o4 += 4)   // MP is a multiple of 4
#pragma unroll
            for (int o = o4; o < o4 + 4; ++o) {
              const float4 v = *reinterpret_cast<const float4*>(ob + o * OS);
              const float2 dx = __fadd2_rn(make_float2(v.x, v.x), make_float2(own[0][0], own[0][1]));
              const float2 dy = __fadd2_rn(make_float2(v.y, v.y), make_float2(own[1][0], own[1][1]));
              float2 q;
              if (ND == 3) {
                const float4 v2 = *reinterpret_cast<const float4*>(ob + o * OS + 4);
                const float2 dz = __fadd2_rn(make_float2(v.z, v.z),
                                             make_float2(own[ND - 1][0], own[ND - 1][1]));
                q = __ffma2_rn(__fmul2_rn(dz, make_float2(v2.x, v2.x)), dz, make_float2(v.w, v.w));
                q = __ffma2_rn(dy, dy, q);
              } else {
                q = __ffma2_rn(dy, dy, make_float2(v.z, v.z));
              }
              q = __ffma2_rn(dx, dx, q);
              mm = push_hit(mm, __float_as_uint(q.x) | __float_as_uint(q.y));
            }
          } else {
            const float* obase = sObs + ((size_t)kg * MP + o0) * ND2;
#pragma unroll 4
            for (int o = 0; o < oc; ++o) {
              const float4 v = *reinterpret_cast<const float4*>(obase + (size_t)o * ND2);
              const float th = sObsThr[o0 + o];
              const float2 dx = __fadd2_rn(make_float2(v.x, v.y), nx);
              const float2 dy = __fadd2_rn(make_float2(v.z, v.w), ny);
              float2 q = __ffma2_rn(dy, dy, make_float2(-th, -th));
              q = __ffma2_rn(dx, dx, q);
              if (ND == 3) {
                const float kp = sObsThr[MP + o0 + o];
                const float4 v2 = *reinterpret_cast<const float4*>(obase + (size_t)o * ND2 + 4);
                const float2 dz = __fadd2_rn(make_float2(v2.x, v2.y), nz);
                q = __ffma2_rn(__fmul2_rn(dz, make_float2(kp, kp)), dz, q);
              }
              mm = push_hit(mm, __float_as_uint(q.x) | __float_as_uint(q.y));
            }
          }
          mask = __brev(mm) >> (32 - oc);
        } else {
          const int ov = max(0, min(32, m - o0));
          mask = (ov >= 32) ? FULL : ((1u << ov) - 1u);
        }
        if (!live) mask = 0u;
        return mask;
      };

      {  // @stage B_pair_exact
        // n <= 32 with static obstacles (one chunk): the exact pair and obstacle rows run in one
        // loop, a lane's pair bits first then its obstacle bits — each lane's order of the
        // two-loop form, in max(pairs + obstacles) instead of max(pairs) + max(obstacles) steps
        const bool merge = merge_rows;
        unsigned pdef = 0u;
        int pj0 = 0;   // first robot of the pair chunk deferred to the merged loop
        // B: robots, in chunks of 32 bodies (one chunk of NJ for n <= 32)
        for (int j0 = 0; j0 < (BIG ? n : 1); j0 += 32) {
          const int jc = BIG ? min(32, n - j0) : n;
          unsigned mask = 0u;
          if (!force) {
            mask = pair_screen(j0, jc);
          } else {
            mask = (jc >= 32) ? FULL : ((1u << jc) - 1u);
          }
          if (i >= j0 && i < j0 + jc) mask &= ~(1u << (i - j0));
          if (!live) mask = 0u;
#ifdef SFB_EXP_NOEXACT
          if (__float_as_uint(own[0][0]) != 0x12345678u) mask = 0u;   // timing ablation only
#endif
          if (P.counters) c_screen += (unsigned)(jc - ((i >= j0 && i < j0 + jc) ? 1 : 0)) * nsteps;
          SFB_TSUB(7);

          // B': exact rows of the flagged partners (warp-uniform loop; shuffles need all lanes)  // @stage B_pair_exact
          if (merge && j0 + 32 >= (BIG ? n : 1)) {   // the last pair chunk joins the obstacle rows
            pdef = mask;
            pj0 = j0;
          }
          else
          while (__any_sync(FULL, mask != 0u)) {
            const bool act = mask != 0u;
            const int jl = act ? __ffs(mask) - 1 : 0;
            mask &= mask - 1u;
            const int j = j0 + jl;
            double pj[ND][2];
            if (TW) {
              const int jj = act ? j : 0;
#pragma unroll
              for (int a = 0; a < ND; ++a) {
                pj[a][0] = tr0[a * CA + (jj ^ sw0)];
                pj[a][1] = tr1[a * CA + (jj ^ sw1)];
              }
            } else if (BIG) {
              const float* hp = sPos + ((size_t)pslot * NROW + (act ? j : 0)) * ND2;
              const float* lp = sLo + ((size_t)pslot * NROW + (act ? j : 0)) * ND2;
              hilo_positions<ND>(hp, lp, pj);
            } else {
              const int src = sub * LW + jl;
#pragma unroll
              for (int a = 0; a < ND; ++a)
#pragma unroll
                for (int kk = 0; kk < 2; ++kk) pj[a][kk] = __shfl_sync(FULL, p[a][kk], src);
            }
            if (act) {
              const double cs = (i < j) ? 1.0 : -1.0;
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                if (kk < nsteps) {
                  double d[ND], r[ND];
#pragma unroll
                  for (int a = 0; a < ND; ++a) d[a] = p[a][kk] - pj[a][kk];
                  ++c_exact;
                  if (row_exact<ND>(d, sKD[KC_INV_A2], sKD[KC_INV_B2], sKD[KC_RA], sKD[KC_RB], sKD[KC_DMAX], cs, r)) {
                    if (i < j) ++c_active;   // each pair row once, like the reference's F rows
                    double rr = 0.0;
#pragma unroll
                    for (int a = 0; a < ND; ++a) {
                      g[a][kk] += r[a];
                      rr = fma(r[a], r[a], rr);
                    }
                    if (i < j) s1 += rr;
                  }
                }
              }
            }
          }
        }

        SFB_TSUB(8);  // @stage B_obs_screen
        // B: obstacles (padded to MP), in chunks of 32
#ifdef SFB_EXP_NOOBS
        for (int o0 = 0; o0 < 0; o0 += 32) {
#else
        for (int o0 = 0; o0 < MP; o0 += 32) {
#endif
          unsigned mask = obs_screen(o0);
#ifdef SFB_EXP_NOEXACT
          if (__float_as_uint(own[0][0]) != 0x12345678u) mask = 0u;
#endif
          if (P.counters) c_screen += (unsigned)max(0, min(32, m - o0)) * nsteps;
          // exact rows of the flagged obstacles; static and moving obstacles in separate loops so  // @stage B_obs_exact
          // the static path issues no (speculative) global load of the track
          auto obs_rows = [&](auto is_static) {
            constexpr bool ST = decltype(is_static)::value;
            while (mask) {
              const int o = o0 + __ffs(mask) - 1;
              mask &= mask - 1u;
              const double4 ax = *reinterpret_cast<const double4*>(sObsAx + 4 * o);
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                if (kk < nsteps) {
                  const int k = 2 * kg + kk;
                  double d[ND], r[ND];
#pragma unroll
                  for (int a = 0; a < ND; ++a)
                    d[a] = p[a][kk] - (ST ? sObsC[o * ND + a] : __ldg(opos + ((size_t)a * m + o) * K1 + k));
                  ++c_exact;
                  if (row_exact<ND>(d, ax.x, ax.y, ax.z, ax.w, sKD[KC_DMAX], 1.0, r)) {
                    ++c_active;
                    double rr = 0.0;
#pragma unroll
                    for (int a = 0; a < ND; ++a) {
                      g[a][kk] += r[a];
                      rr = fma(r[a], r[a], rr);
                    }
                    s1 += rr;
                  }
                }
              }
            }
          };
          if (merge) {
            // one loop over a lane's pair bits, then its obstacle bits; the body is branch-free
            // apart from the row math's rare slow path (partner position and row parameters
            // by select), so a pass costs the same for pair and obstacle rows
            unsigned pmk = pdef, omk = mask;
            const int tb0 = P.L.gl / 8 + k0 * TS, tb1 = P.L.gl / 8 + k1 * TS, ob0 = P.L.obs_c / 8;
            const uint32_t sbase = smem_u32(smem);
            // TBL: a partner robot's exact positions come from the table (phase A), so each
            // lane runs its own rows without warp-synchronous exchanges; obstacle centres and
            // axes from shared memory (the pair axes are the double4 at sKD[KC_INV_A2])
            // (n > 32: partner positions from the FP32 hi/lo rows, also per lane)
            while ((TBL || BIG) ? ((pmk | omk) != 0u) : __any_sync(FULL, (pmk | omk) != 0u)) {
              const bool isp = pmk != 0u;
              const bool act = isp || omk != 0u;
              const int bit = __ffs(isp ? pmk : omk) - 1;          // -1: no row left
              pmk = isp ? (pmk & (pmk - 1u)) : pmk;
              omk = isp ? omk : (omk & (omk - 1u));
              const int jl = isp ? bit : 0, o = isp ? 0 : max(bit, 0);
              double pj[ND][2];
              if (TBL) {
                // 32-bit shared-window addresses selected per row kind
#pragma unroll
                for (int a = 0; a < ND; ++a) {   // (in this per-lane loop bit >= 0)
                  const int q0 = isp ? tb0 + a * CA + (bit ^ sw0) : ob0 + bit * ND + a;
                  const int q1 = isp ? tb1 + a * CA + (bit ^ sw1) : q0;
                  pj[a][0] = lds_f64(sbase + 8 * q0);
                  pj[a][1] = lds_f64(sbase + 8 * q1);
                }
              } else if (BIG) {
                if (isp && TW) {
#pragma unroll
                  for (int a = 0; a < ND; ++a) {
                    pj[a][0] = tr0[a * CA + ((pj0 + jl) ^ sw0)];
                    pj[a][1] = tr1[a * CA + ((pj0 + jl) ^ sw1)];
                  }
                } else if (isp) {
                  const float* hp = sPos + ((size_t)pslot * NROW + pj0 + jl) * ND2;
                  const float* lp = sLo + ((size_t)pslot * NROW + pj0 + jl) * ND2;
                  hilo_positions<ND>(hp, lp, pj);
                } else {
#pragma unroll
                  for (int a = 0; a < ND; ++a) pj[a][0] = pj[a][1] = sObsC[o * ND + a];
                }
              } else {
                if (__any_sync(FULL, isp)) {
                  const int src = sub * LW + jl;
#pragma unroll
                  for (int a = 0; a < ND; ++a)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) pj[a][kk] = __shfl_sync(FULL, p[a][kk], src);
                }
                if (!isp) {
#pragma unroll
                  for (int a = 0; a < ND; ++a) pj[a][0] = pj[a][1] = sObsC[o * ND + a];
                }
              }
              double ia2, ib2, aa, bb;
              if (TBL) {
                const uint32_t axa = sbase + (isp ? P.L.kc + KC_INV_A2 * 8 : P.L.obs_ax + 32 * bit);
                const double2 a01 = lds_f64x2(axa), a23 = lds_f64x2(axa + 16);
                ia2 = a01.x; ib2 = a01.y; aa = a23.x; bb = a23.y;
              } else {
                const double4 ax = *reinterpret_cast<const double4*>(isp ? sKD + KC_INV_A2 : sObsAx + 4 * o);
                ia2 = ax.x; ib2 = ax.y; aa = ax.z; bb = ax.w;
              }
              const bool once = !isp || i < pj0 + (TBL ? bit : jl);   // rows the reference's F holds once
              const double cs = once ? 1.0 : -1.0;
#pragma unroll
              for (int kk = 0; kk < 2; ++kk) {
                if (act && kk < nsteps) {
                  double d[ND], r[ND];
#pragma unroll
                  for (int a = 0; a < ND; ++a) d[a] = p[a][kk] - pj[a][kk];
                  ++c_exact;
                  if (row_exact<ND>(d, ia2, ib2, aa, bb, sKD[KC_DMAX], cs, r)) {
                    double rr = 0.0;
#pragma unroll
                    for (int a = 0; a < ND; ++a) {
                      g[a][kk] += r[a];
                      rr = fma(r[a], r[a], rr);
                    }
                    if (once) {
                      ++c_active;
                      s1 += rr;
                    }
                  }
                }
              }
            }
          } else if (P.obs_static) {
            obs_rows(std::true_type{});
          } else {
            obs_rows(std::false_type{});
          }
        }

      }

      SFB_TSUB(9);
      // B": workspace box rows (exact). Compact mode first tests the FP32 positions against
      // the box shrunk by bmg (>> their rounding error below plim): a warp whose positions are
      // all strictly inside skips the rows, which are then exactly zero.
      bool box_rows = true;
      if (compact && !force) {
        // per axis: the larger / smaller of the lane's steps against the shrunk box (a missing
        // second step repeats the first; a lane without steps is never out). NaN positions
        // need no rows here: the FP64 rows below add nothing for them either.
        bool out = false;
#pragma unroll
        for (int a = 0; a < ND; ++a) {
          const float v1 = has1 ? own[a][1] : own[a][0];
          out |= (fmaxf(own[a][0], v1) > sKF[KC_F_BHI + a]) | (fminf(own[a][0], v1) < sKF[KC_F_BLO + a]);
        }
        box_rows = __any_sync(FULL, live && out);
      }  // @stage box
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        if (box_rows && kk < nsteps) {
#pragma unroll
          for (int a = 0; a < ND; ++a) {
            const double up = p[a][kk] - sKD[KC_BHI + a];
            const double lo = sKD[KC_BLO + a] - p[a][kk];
            if (up > 0.0) { g[a][kk] += up; s2 = fma(up, up, s2); }
            if (lo > 0.0) { g[a][kk] -= lo; s2 = fma(lo, lo, s2); }
          }
        }
      }

      // C: TBL stores g_i(k) for the tensor-core contraction after the task loop; otherwise
      // contraction with W^T into the lane's partial G  // @stage C_contract
      if (TAB) {
        // every lane's rows have read the partner positions of these steps (TW: the rows of the
        // k-group's other robot blocks too)
        if (TW) asm volatile("bar.sync %0, %1;" ::"r"(1 + wk), "r"(P.RB * 32) : "memory");
        else __syncwarp();
        if (live) {
          double* w0 = const_cast<double*>(tr0);
          double* w1 = const_cast<double*>(tr1);
#pragma unroll
          for (int a = 0; a < ND; ++a) {
            w0[a * CA + (i ^ sw0)] = g[a][0];
            if (has1) w1[a * CA + (i ^ sw1)] = g[a][1];
          }
        }
      } else if (__any_sync(FULL, nsteps > 0)) {
#pragma unroll
        for (int c = 0; c < NXI; ++c) {
          const double2 w = make_double2(w0r[c], w1r[c]);
#pragma unroll
          for (int a = 0; a < ND; ++a) {
            if (a < RA) {
              double& acc = Gp[a < RA ? a : 0][c];
              acc = fma(w.x, g[a][0], fma(w.y, g[a][1], acc));
            } else {
              double* q = gl + (c * ND + a) * 32;
              *q = fma(w.x, g[a][0], fma(w.y, g[a][1], *q));
            }
          }
        }
      }
      __syncwarp();   // the next task overwrites this warp's position row
      SFB_TSUB(10);
    }

    // -------------------------------------------- reductions  // @stage G_reduce
    // TBL: the KKT's boundary-row columns u = b - E xi (xi is the iterate of this iteration
    // and stays fixed until E2) are computed here by the warps that ran fewer k-group tasks,
    // while the others finish theirs; E1 then only has the Delta columns
    double equ = 0.0;
    if (TBL) {
      const int ncu = ND * NB, ntask = ts_hi - ts_lo, R = ntask % nw, Lw = nw - R;
      int t0 = warp, dt = nw;                       // spread over every warp ...
      if (R != 0 && (Lw >= 4 || ntask < nw)) {      // ... or over the lighter ones (in cluster
        t0 = warp >= R ? warp - R : ncu;            // mode, the warps that had no task at all)
        dt = Lw;
      }
      // UCB columns per pass with independent chains (the per-column arithmetic and the xor
      // tree are unchanged: same bits)
      constexpr int UCB = 4;
      for (int tb = t0; tb < ncu; tb += UCB * dt) {
        double csum[UCB];
#pragma unroll
        for (int q = 0; q < UCB; ++q) {           // loads and arithmetic first ...
          const int t = tb + q * dt;
          csum[q] = 0.0;
          if (t < ncu && lane < n) {
            const int a = (t >= NB) + (ND == 3 && t >= 2 * NB), r = t - a * NB;
            const int ai = a * n + lane;
            const double* x = sXi + ai * NXP;
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < NXI; ++c) v = fma(sE[r * NXI + c], x[c], v);
            const double u = __ldg(gBv + ai * NB + r) - v;
            equ = fmax(equ, fabs(u));
            csum[q] = u;
          }
        }
#pragma unroll
        for (int q = 0; q < UCB; ++q) {           // ... then the stores
          const int t = tb + q * dt;
          if (t < ncu && lane < n) {
            const int a = (t >= NB) + (ND == 3 && t >= 2 * NB), r = t - a * NB;
            sU[(a * n + lane) * NB + r] = csum[q];
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int q = 0; q < UCB; ++q) csum[q] += __shfl_xor_sync(FULL, csum[q], off);
        if (lane == 0) {
#pragma unroll
          for (int q = 0; q < UCB; ++q)
            if (tb + q * dt < ncu) sSU[tb + q * dt] = csum[q];
        }
      }
    }
    if (!BIG && RA > 0) {
#pragma unroll
      for (int a = 0; a < (RA > 0 ? RA : 1); ++a)
#pragma unroll
        for (int c = 0; c < NXI; ++c) gl[(c * ND + a) * 32] = Gp[a][c];
    }
    // fpp: the previous iteration's per-lane fixed-point partial, reduced here next to s1, s2
    // (its xor tree used to end the KKT step on the serial path; same tree, same value)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      s1 += __shfl_xor_sync(FULL, s1, off);
      s2 += __shfl_xor_sync(FULL, s2, off);
      fpp += __shfl_xor_sync(FULL, fpp, off);
    }
    if (lane == 0) {
      sRed[warp * 4 + 0] = s1;
      sRed[warp * 4 + 1] = s2;
      sRed[warp * 4 + 3] = fpp;
    }
    SFB_TMARK(0);
    __syncthreads();   // all positions consumed: the union region is free
    SFB_TMARK(1);
#ifdef SFB_PHASE_TIMING
    if (tid == 0) t_sub = clock64();
#endif

    if (TAB) {
      // G^T (c x col) = W^T (c x k) . g (k x col) on the FP64 tensor cores (DMMA m8n8k4): warp
      // per 8-column tile, two 8-row tiles of c, k in steps of 4 over this CTA's steps [klo, khi)
      // (rows outside are masked, never read), even/odd k-steps in separate accumulators then
      // added: a fixed order, deterministic. A(m = c, k) = W[k][c], B(k, col) = g[k][col].
      const int ncol = ND * CA, ntl = ncol >> 3;         // table columns a * CA + i
      const int klo = 2 * SUB * ts_lo, khi = min(K1, 2 * SUB * ts_hi);
      const int rq = lane >> 2, kq = lane & 3;
      for (int tl = warp; tl < ntl; tl += nw) {
        double acc[2][2][2];   // [parity][m tile][2]
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) acc[q2][mt][0] = acc[q2][mt][1] = 0.0;
        const int colB = tl * 8 + rq;
        const bool colok = colB < ncol;
        if (klo == 0 && khi == K1) {
          // whole time axis: rows K1.. of the table and of W are zero, columns beyond the live
          // ones only feed output rows/columns that are not stored: no masks
          const double* tb = sTab + (size_t)kq * TS + (colB ^ tab_swz(kq));   // k & 3 == kq
          const double* wa = sW + (size_t)kq * WSTR + rq;
          const int nks = (K1 + 3) >> 2;
          int ks = 0;
          for (; ks + 1 < nks; ks += 2) {
#pragma unroll
            for (int q2 = 0; q2 < 2; ++q2) {
              const double bv = tb[(size_t)(4 * (ks + q2)) * TS];
              const double a0 = wa[(size_t)(4 * (ks + q2)) * WSTR], a1 = wa[(size_t)(4 * (ks + q2)) * WSTR + 8];
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(acc[q2][0][0]), "+d"(acc[q2][0][1]) : "d"(a0), "d"(bv));
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(acc[q2][1][0]), "+d"(acc[q2][1][1]) : "d"(a1), "d"(bv));
            }
          }
          if (ks < nks) {
            const double bv = tb[(size_t)(4 * ks) * TS];
            const double a0 = wa[(size_t)(4 * ks) * WSTR], a1 = wa[(size_t)(4 * ks) * WSTR + 8];
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[0][0][0]), "+d"(acc[0][0][1]) : "d"(a0), "d"(bv));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[0][1][0]), "+d"(acc[0][1][1]) : "d"(a1), "d"(bv));
          }
        } else
        for (int ks = klo >> 2; ks < (khi + 3) >> 2; ks += 2) {
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {
            const int k = 4 * (ks + q2) + kq;
            const bool kin = k >= klo && k < khi;
            const double bv = (kin && colok) ? sTab[(size_t)k * TS + (colB ^ tab_swz(k))] : 0.0;
            const double* wk = sW + (size_t)k * WSTR;      // zero padded beyond NXI
            const double a0 = kin ? wk[rq] : 0.0;
            const double a1 = (kin && 8 + rq < NXI) ? wk[8 + rq] : 0.0;
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[q2][0][0]), "+d"(acc[q2][0][1]) : "d"(a0), "d"(bv));
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[q2][1][0]), "+d"(acc[q2][1][1]) : "d"(a1), "d"(bv));
          }
        }
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const int c = mt * 8 + rq;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int col = tl * 8 + kq * 2 + j;
            if (c < NXI && (col & (CA - 1)) < n) sG[((col / CA) * n + (col & (CA - 1))) * NXI + c] = acc[0][mt][j] + acc[1][mt][j];
          }
        }
      }
      SFB_TSUB(16);
      __syncthreads();
    } else if (!BIG) {
      // G = sum over warps, then over the k-group sub-lanes, of the per-lane partials (fixed order)
      // thread = (column (c, a), robot): consecutive threads read consecutive lanes
      for (int o = tid; o < NXI * ND * 32; o += nt) {
        const int ii = o & 31, col = o >> 5;
        if (ii >= n) continue;
        const int c = col / ND, a = col - c * ND;
        double v[NW * SUB];
#pragma unroll
        for (int w = 0; w < NW; ++w)
#pragma unroll
          for (int s2i = 0; s2i < SUB; ++s2i)
            v[w * SUB + s2i] = w < nw ? sGl[(size_t)(w * NXI * ND + col) * 32 + ii + s2i * NJ] : 0.0;
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < NW * SUB; ++q) acc += v[q];
        sG[(a * n + ii) * NXI + c] = acc;
      }
      __syncthreads();
    }
    // n > 32: G partials in slots; slot s of round r holds warp r*slots + s, layout [ND][32][NXI]
    const int slots = P.L.slots;
    for (int w0 = 0; BIG && !TW && w0 < nw; w0 += slots) {
      if (warp >= w0 && warp < w0 + slots && robot_ok) {
        double* dst = sSlot + (size_t)(warp - w0) * ND * 32 * NXI;
#pragma unroll
        for (int a = 0; a < (BIG ? ND : 1); ++a)
#pragma unroll
          for (int c = 0; c < (BIG ? NXI : 1); ++c) dst[(a * 32 + lane) * NXI + c] = Gp[BIG ? a : 0][BIG ? c : 0];
      }
      __syncthreads();
      for (int o = tid; o < nv; o += nt) {
        int ai, c, a, ii;
        split(o, ai, c, a, ii);
        const int rbi = ii >> 5, li = ii & 31;
        double acc = (w0 == 0) ? 0.0 : sG[o];
        const int wend = min(nw, w0 + slots);
        for (int w = w0; w < wend; ++w) {
          if ((BIG ? (w & (P.RB - 1)) : 0) != rbi) continue;
          acc += sSlot[(size_t)(w - w0) * ND * 32 * NXI + (a * 32 + li) * NXI + c];
        }
        sG[o] = acc;
      }
      __syncthreads();
    }

    SFB_TMARK(2);
    // -------------------------------------------- D: residuals, trace, convergence  // @stage D_decision
    double S1 = 0.0, S2 = 0.0, FP = 0.0;
#pragma unroll
    for (int w = 0; w < MW; ++w) {
      if (w >= nw) break;
      S1 += sRed[w * 4 + 0];
      S2 += sRed[w * 4 + 1];
      FP += sRed[w * 4 + 3];
    }
    if (csize > 1) {
      // Cluster reduction of the CTA partials (G and S1, S2) in two DSMEM pushes, each
      // completing on the receiver's mbarrier (st.async ... complete_tx):
      //  1. reduce-scatter: slice s of the partial goes to rank s's receive buffer,
      //  2. rank s sums its slice over the ranks in rank order and stores the sum into every
      //     rank's G (whose local partial was already scattered in step 1).
      // No cluster barrier is needed to reuse a buffer: a rank's next push into it depends on
      // data the buffer's owner sends only after it has consumed the buffer.
      const uint32_t par = (uint32_t)(it & 1);
      auto slice_len = [&](int r) { return max(0, min(xSL, xtot - r * xSL)); };
      if (tid == 0) {
        sG[nv] = S1;
        sG[nv + 1] = S2;
        if (xtot > nv + 2) sG[nv + 2] = 0.0;
        mbar_expect_tx(xbar1, (uint32_t)(csize * slice_len(crank) * 8));
      }
      __syncthreads();
#ifdef SFB_PHASE_TIMING
      if (tid == 0) t_sub = clock64();
#endif
      SFB_JITTER(3, it);
      for (int o = 2 * tid; o < xtot; o += 2 * nt) {
        const int sr = o / xSL;
        st_async_v2(dsmem_map(smem_u32(xrecv + (size_t)crank * xSL + (o - sr * xSL)), sr), sG[o], sG[o + 1],
                    dsmem_map(xbar1, sr));
      }
      SFB_JITTER(4, it);
      mbar_wait(xbar1, par);
      SFB_JITTER(5, it);
      SFB_TSUB(11);
      if (tid == 0) mbar_expect_tx(xbar2, (uint32_t)(xtot * 8));
      const int mylen = slice_len(crank);
      for (int j = 2 * tid; j < mylen; j += 2 * nt) {
        double a0 = 0.0, a1 = 0.0;
        for (int r = 0; r < csize; ++r) {
          a0 += xrecv[(size_t)r * xSL + j];
          a1 += xrecv[(size_t)r * xSL + j + 1];
        }
        const uint32_t dst = smem_u32(sG + crank * xSL + j);
        for (int r = 0; r < csize; ++r) st_async_v2(dsmem_map(dst, r), a0, a1, dsmem_map(xbar2, r));
      }
      SFB_JITTER(6, it);
      mbar_wait(xbar2, par);
      SFB_TSUB(12);
      S1 = sG[nv];
      S2 = sG[nv + 1];
      SFB_TSUB(13);
    }
    const double primal = sqrt(S1) + sqrt(S2);
    if (it > 0) last_fp = FP;
    ++c_evals;
    if (tid == 0 && crank == 0 && P.trace) {
      double* tr = P.trace + ((size_t)member() * (P.max_iters + 1) + it) * 2;
      tr[0] = primal;
      tr[1] = last_fp;
    }
    const bool conv_p = P.early_exit && (primal < P.primal_tol) && it >= 1;
    const bool conv_f = P.early_exit && (last_fp < P.fp_tol);
    if (conv_p || conv_f || it == P.max_iters) {
      // the xi committed at it-1 has not had its boundary residual measured yet
      if (it > 0) {
        double eqp = eql;   // this lane's running max over the earlier committed steps
        for (int ai = tid; ai < nrows; ai += nt) {
          const double* x = sXi + ai * NXP;
          for (int r = 0; r < NB; ++r) {
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < NXI; ++c) v = fma(sE[r * NXI + c], x[c], v);
            eqp = fmax(eqp, fabs(v - __ldg(gBv + ai * NB + r)));
          }
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) eqp = fmax(eqp, __shfl_xor_sync(FULL, eqp, off));
        if (lane == 0) sRed[warp * 4 + 2] = eqp;
        __syncthreads();
        #pragma unroll
        for (int w = 0; w < MW; ++w)
          if (w < nw) eq_max = fmax(eq_max, sRed[w * 4 + 2]);
      }
      double* xo = P.xi + (size_t)member() * nv;
      double* lo = P.lam + (size_t)member() * nv;
      for (int o = tid; crank == 0 && o < nv; o += nt) {
        const int ai = o / NXI, c = o - ai * NXI;
        xo[o] = sXi[ai * NXP + c];
        lo[o] = sLam[ai * NXP + c];
      }
      if (tid == 0 && crank == 0) {
        P.primal[member()] = primal;
        P.eq_max[member()] = eq_max;
        P.iterations[member()] = it;
        P.status[member()] = conv_p ? 1 : (conv_f ? 2 : 0);
      }
      break;
    }

    SFB_TMARK(3);
#ifdef SFB_PHASE_TIMING
    if (tid == 0) t_sub = clock64();
#endif
    // -------------------------------------------- E: multiplier update and KKT step  // @stage E1_kkt
    // E1: one warp per column, lanes = robots. Columns (a, c): lambda+, Delta and the robot
    // sum of Delta; columns (a, r): u = b - E xi, its robot sum, and max|u| (the boundary
    // residual of the xi committed at it-1, solver.py:336-337). Sums use a fixed xor tree.
    fpp = 0.0;
    const int ncolD = ND * NXI, ncol = ncolD + (TBL ? 0 : ND * NB);
    // UC1 columns per pass (warp w: columns w, w + nw, ... in that order), independent chains;
    // the per-column arithmetic, the fpp order and the xor tree are unchanged
    constexpr int UC1 = 3;
    for (int cb = warp; cb < ncol; cb += UC1 * nw) {
     double csumv[UC1];
#pragma unroll
     for (int q = 0; q < UC1; ++q) {
      const int col = cb + q * nw;
      double csum = 0.0;
      if (col >= ncol) {
      } else if (col < ncolD) {
        const int a = col / NXI, c = col - a * NXI;
        for (int i0 = 0; i0 < (BIG ? n : 1); i0 += 32) {   // n <= 32: one pass
          const int ii = i0 + lane;
          if (ii < n) {
            const int ai = a * n + ii;
            const double lo = sLam[ai * NXP + c];
            const double ln = fma(-P.rho, sG[ai * NXI + c], lo);
            double qx;
            if (P.mode == 0) {
              qx = sXi[ai * NXP + c];
            } else {
              qx = 0.0;
              const double* x = sXi + ai * NXP;
#pragma unroll
              for (int c2 = 0; c2 < NXI; ++c2) qx = fma(sQ[c * NXI + c2], x[c2], qx);
            }
            const double t = sTgt[ai * NXI + c];
            const double d = 2.0 * ln - lo + t - qx;
            sD[ai * NXI + c] = d;
            sLam[ai * NXP + c] = ln;
            const double dl = ln - lo;
            fpp = fma(dl, dl, fpp);
            csum += d;
          }
        }
      } else {
        const int t2 = col - ncolD, a = (t2 >= NB) + (ND == 3 && t2 >= 2 * NB), r = t2 - a * NB;
        for (int i0 = 0; i0 < (BIG ? n : 1); i0 += 32) {   // n <= 32: one pass
          const int ii = i0 + lane;
          if (ii < n) {
            const int ai = a * n + ii;
            const double* x = sXi + ai * NXP;
            double v = 0.0;
#pragma unroll
            for (int c = 0; c < NXI; ++c) v = fma(sE[r * NXI + c], x[c], v);
            const double u = __ldg(gBv + ai * NB + r) - v;
            sU[ai * NB + r] = u;
            equ = fmax(equ, fabs(u));
            csum += u;
          }
        }
      }
      csumv[q] = csum;
     }
#pragma unroll
     for (int off = 16; off > 0; off >>= 1)
#pragma unroll
       for (int q = 0; q < UC1; ++q) csumv[q] += __shfl_xor_sync(FULL, csumv[q], off);
     if (lane == 0) {
#pragma unroll
       for (int q = 0; q < UC1; ++q) {
         const int col = cb + q * nw;
         if (col < ncolD) sSD[col] = csumv[q];
         else if (col < ncol) sSU[col - ncolD] = csumv[q];
       }
     }
    }
    SFB_TSUB(17);
    // boundary residual max over committed steps: a per-lane running max, reduced over the CTA
    // once at exit (max is order-free: the same value as a per-iteration reduction)
    if (it > 0) eql = fmax(eql, equ);
    __syncthreads();
    SFB_TMARK(4);
#ifdef SFB_PHASE_TIMING
    if (tid == 0) t_sub = clock64();
#endif
    // E2: xi+ = xi + Pxx Delta_i + Pxb u_i + (Dxx sum Delta + Dxb sum u)  // @stage E2_kkt
#ifndef SFB_E2_SIMT
#define SFB_E2_SIMT 0   // experiments: 1 runs the SIMT xi update also on the TBL path
#endif
    if (TBL && !SFB_E2_SIMT) {
      // on the FP64 tensor cores: X+ (rows x c) = (X + mean) + [Delta | u] (rows x (NXI + NB))
      // . [Pxx | Pxb]^T, warp per 8-row tile, two 8-column tiles, k in steps of 4 (DMMA m8n8k4).
      // mean[a][c] is computed by lane a * NXI + c (and + 32) and fetched by shuffle.
      const int KT = NXI + NB, nrow = ND * n, nmt = (nrow + 7) >> 3;
      const int rq = lane >> 2, kq = lane & 3;
      double mv[(ND * NXI + 31) / 32];
#pragma unroll
      for (int h = 0; h < (ND * NXI + 31) / 32; ++h) {
        const int idx = lane + 32 * h;
        double m0 = 0.0, m1 = 0.0;
        if (idx < ND * NXI) {
          const int a = idx / NXI, c = idx - a * NXI;
#pragma unroll
          for (int c2 = 0; c2 < NXI; ++c2) m0 = fma(sDxx[c * NXI + c2], sSD[a * NXI + c2], m0);
#pragma unroll
          for (int r = 0; r < NBM; ++r)
            if (r < NB) m1 = fma(sDxb[c * NB + r], sSU[a * NB + r], m1);
        }
        mv[h] = m0 + m1;
      }
      SFB_TSUB(14);
      for (int tl = warp; tl < nmt; tl += nw) {
        const int row = tl * 8 + rq;
        const bool rowok = row < nrow;
        const int ra = (row >= n) + (ND == 3 && row >= 2 * n);
        double acc[2][2];
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = nt2 * 8 + 2 * kq + j;
            const int idx = ra * NXI + c;
            double mval = 0.0;
#pragma unroll
            for (int h = 0; h < (ND * NXI + 31) / 32; ++h) {
              const double v = __shfl_sync(FULL, mv[h], idx & 31);
              if ((idx >> 5) == h) mval = v;
            }
            acc[nt2][j] = (rowok && c < NXI) ? sXi[row * NXP + c] + mval : 0.0;
          }
        // all fragments first (no branches between the loads), then the DMMA chain; the
        // operands and the k order are those of the per-step form (same bits)
        constexpr int KSM = (NXI + NBM + 3) / 4;
        const int nks = (KT + 3) >> 2;
        double av[KSM], bv[KSM][2];
#pragma unroll
        for (int ks = 0; ks < KSM; ++ks) {
          const int k = 4 * ks + kq;
          const double* ap = (k < NXI) ? sD + row * NXI + k : sU + row * NB + (k - NXI);
          av[ks] = (rowok && k < KT) ? *ap : 0.0;
          bv[ks][0] = ks < nks ? sPB[(ks * 2) * 32 + lane] : 0.0;
          bv[ks][1] = ks < nks ? sPB[(ks * 2 + 1) * 32 + lane] : 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < KSM; ++ks) {
          if (ks < nks) {
#pragma unroll
            for (int nt2 = 0; nt2 < 2; ++nt2)
              asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                           : "+d"(acc[nt2][0]), "+d"(acc[nt2][1]) : "d"(av[ks]), "d"(bv[ks][nt2]));
          }
        }
#pragma unroll
        for (int nt2 = 0; nt2 < 2; ++nt2)
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = nt2 * 8 + 2 * kq + j;
            if (rowok && c < NXI) {
              const double xo = sXi[row * NXP + c];
              const double xn = acc[nt2][j];
              sXi[row * NXP + c] = xn;
              const double dx = xn - xo;
              fpp = fma(dx, dx, fpp);
            }
          }
      }
      SFB_TSUB(15);
    } else
    for (int col = warp; col < ncolD; col += nw) {
      const int a = col / NXI, c = col - a * NXI;
      double m0 = 0.0, m1 = 0.0;
#pragma unroll
      for (int c2 = 0; c2 < NXI; ++c2) m0 = fma(sDxx[c * NXI + c2], sSD[a * NXI + c2], m0);
#pragma unroll
      for (int r = 0; r < NBM; ++r)
        if (r < NB) m1 = fma(sDxb[c * NB + r], sSU[a * NB + r], m1);
      const double mean = m0 + m1;
      for (int i0 = 0; i0 < (BIG ? n : 1); i0 += 32) {   // n <= 32: one pass
        const int ii = i0 + lane;
        if (ii < n) {
          const int ai = a * n + ii;
          const double* dv = sD + ai * NXI;
          const double* uv = sU + ai * NB;
          double acc0 = 0.0, acc1 = 0.0;
#pragma unroll
          for (int c2 = 0; c2 + 1 < NXI; c2 += 2) {
            acc0 = fma(sPxx[c * NXI + c2], dv[c2], acc0);
            acc1 = fma(sPxx[c * NXI + c2 + 1], dv[c2 + 1], acc1);
          }
          if (NXI & 1) acc0 = fma(sPxx[c * NXI + NXI - 1], dv[NXI - 1], acc0);
#pragma unroll
          for (int r = 0; r < NBM; ++r)
            if (r < NB) acc1 = fma(sPxb[c * NB + r], uv[r], acc1);
          const double xo = sXi[ai * NXP + c];
          const double xn = xo + ((acc0 + acc1) + mean);
          sXi[ai * NXP + c] = xn;
          const double dx = xn - xo;
          fpp = fma(dx, dx, fpp);
        }
      }
    }
    __syncthreads();
    SFB_JITTER(7, it);
    SFB_TMARK(5);
  }
#ifdef SFB_PHASE_TIMING  // @stage epilogue
  if (tid == 0 && P.counters) {
    for (int q = 0; q < 18; ++q) P.counters[(size_t)member() * 24 + 4 + q] = (unsigned long long)t_ph[q];
  }
#endif

  if (P.counters) {
    unsigned long long w_exact = c_exact, w_active = c_active, w_screen = c_screen;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      w_exact += __shfl_xor_sync(FULL, w_exact, off);
      w_active += __shfl_xor_sync(FULL, w_active, off);
      w_screen += __shfl_xor_sync(FULL, w_screen, off);
    }
    if (lane == 0) {
#ifdef SFB_PHASE_TIMING
      unsigned long long* cb = P.counters + (size_t)member() * 24;
#else
      unsigned long long* cb = P.counters + (size_t)member() * 4;
#endif
      atomicAdd(cb + 0, w_exact);
      atomicAdd(cb + 1, w_active);
      atomicAdd(cb + 2, w_screen);
      if (warp == 0 && crank == 0) atomicAdd(cb + 3, (unsigned long long)c_evals);
    }
  }
  return finished;
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// MW = 16: the capped n > 32 build with 16-warp CTAs, one per SM (small batches and n = 65..128,
// whose layout does not fit half an SM)
template <int ND, int NXI, int NJ, bool BIG, bool BIG2 = false, int MW = NW, bool TW = false>
__global__ void __launch_bounds__(MW * 32, BIG ? (BIG2 ? (MW > NW ? 1 : 2) : 1) : SFB_MINB)
    sf_solve_kernel(const KParams P) {
  // Split schedule ("stream-K" over evaluation units): with B > G resident CTAs, one CTA per
  // member would leave the last of ceil(B / G) waves partly idle (C3: 512 members on 296
  // slots = 1.73 waves of work in 2). Instead the G CTAs form one cooperative wave and CTA c
  // runs units [c U / G, (c + 1) U / G), U = B E, E = max_iters + 1. Since B >= G every range
  // holds at least E units, so at most two members are cut: the range's LAST member (its
  // head, evaluations [0, rb)) runs FIRST and is handed to CTA c + 1, whose range starts
  // with that member's tail, run LAST — by then the head (started at time 0 and no longer
  // than a range) is done, so a CTA does not wait in a balanced wave. Every evaluation runs
  // the same code on the same state, so results are bitwise those of the unsplit launch.
  // Pieces of this CTA in order: [head of mb] [full members] [tail of ma]; one call site of
  // the (large, inlined) member solve.
  // The piece schedule is recomputed per piece (a few integer ops) rather than kept in
  // registers across the member solve (split_build: which builds run it; sfb_solve knows).
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned* sched = reinterpret_cast<unsigned*>(smem + P.L.red + NW_RED * 4 * 8);
  if (!split_build<ND, BIG, BIG2>() || !P.split) {
    if (threadIdx.x == 0) sched[SCHED_MEMBER] = blockIdx.x / P.csize;
    __syncthreads();
    sf_member<ND, NXI, NJ, BIG, BIG2, MW, TW>(P, 0, PIECE_WHOLE, 0);
    return;
  }
  if (threadIdx.x == 0) sched[SCHED_PIECE] = 0u;
  __syncthreads();
  for (;;) {
    const int pc = (int)*reinterpret_cast<volatile unsigned*>(sched + SCHED_PIECE);
    int b = 0, it0 = 0, piece = PIECE_WHOLE, stop = 0;
    {
      const long long E = (long long)P.max_iters + 1, U = (long long)P.B * E, G = gridDim.x;
      const long long c = blockIdx.x, lo = c * U / G, hi = (c + 1) * U / G;
      const int ma = (int)(lo / E), ra = (int)(lo % E), mb = (int)(hi / E), rb = (int)(hi % E);
      const int first = ra ? ma + 1 : ma;
      const int npieces = (rb ? 1 : 0) + (mb - first) + (ra ? 1 : 0);
      if (pc >= npieces) break;
      if (rb && pc == 0) {                        // head of mb, handed to CTA c + 1
        b = mb;
        piece = PIECE_HEAD;
        stop = rb;
      } else if (ra && pc == npieces - 1) {       // tail of ma, from CTA c - 1
        b = ma;
        it0 = ra;
        piece = PIECE_TAIL;
        unsigned f = 0u;
        if (threadIdx.x == 0) {
          while ((f = ld_acquire_gpu(P.hand_flag + c - 1)) == 0u) __nanosleep(256);
          SFB_CHECK(f == 1u || f == 2u);
        }
        // the member may have converged inside the head: nothing left to do
        if (__syncthreads_or(f == 2u)) {
          if (threadIdx.x == 0) sched[SCHED_PIECE] = pc + 1;
          __syncthreads();
          continue;
        }
      } else {
        b = first + pc - (rb ? 1 : 0);
      }
    }
    if (threadIdx.x == 0) sched[SCHED_MEMBER] = b;
    __syncthreads();
    const bool fin = sf_member<ND, NXI, NJ, BIG, BIG2, MW, TW>(P, it0, piece, stop);
    __syncthreads();                              // shared memory reused by the next piece; handoff stores issued
    if (threadIdx.x == 0) {
      const int pcn = (int)sched[SCHED_PIECE];
      if (pcn == 0) {
        const long long E = (long long)P.max_iters + 1, U = (long long)P.B * E;
        if (((long long)blockIdx.x + 1) * U / gridDim.x % E != 0) {   // this was a head piece
          SFB_JITTER(8, pcn);
          __threadfence();
          SFB_CHECK(ld_acquire_gpu(P.hand_flag + blockIdx.x) == 0u);   // each slot handed over once
          st_release_gpu(P.hand_flag + blockIdx.x, fin ? 2u : 1u);
        }
      }
      sched[SCHED_PIECE] = pcn + 1;
    }
    __syncthreads();
  }
}

using KernelFn = void (*)(const KParams);

}  // namespace sfb
