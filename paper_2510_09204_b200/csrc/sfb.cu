// sfb.cu — C ABI (include/sfb.h) of the B200 SF solver: host-side plan (the
// Kronecker-compressed KKT inverse, FP64) and the launch of the persistent kernel.
#include "../../include/sfb.h"
#include "sfb_kernel.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace sfb;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(SFB_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------- host FP64 linear algebra
// Gauss-Jordan inverse with partial pivoting; returns false if singular.
bool invert(std::vector<double> a, int N, std::vector<double>& inv) {
  inv.assign((size_t)N * N, 0.0);
  for (int i = 0; i < N; ++i) inv[(size_t)i * N + i] = 1.0;
  for (int col = 0; col < N; ++col) {
    int piv = col;
    double best = std::fabs(a[(size_t)col * N + col]);
    for (int r = col + 1; r < N; ++r) {
      const double v = std::fabs(a[(size_t)r * N + col]);
      if (v > best) { best = v; piv = r; }
    }
    if (!(best > 0.0)) return false;
    if (piv != col) {
      for (int c = 0; c < N; ++c) {
        std::swap(a[(size_t)piv * N + c], a[(size_t)col * N + c]);
        std::swap(inv[(size_t)piv * N + c], inv[(size_t)col * N + c]);
      }
    }
    const double d = a[(size_t)col * N + col];
    for (int c = 0; c < N; ++c) {
      a[(size_t)col * N + c] /= d;
      inv[(size_t)col * N + c] /= d;
    }
    for (int r = 0; r < N; ++r) {
      if (r == col) continue;
      const double f = a[(size_t)r * N + col];
      if (f == 0.0) continue;
      for (int c = 0; c < N; ++c) {
        a[(size_t)r * N + c] -= f * a[(size_t)col * N + c];
        inv[(size_t)r * N + c] -= f * inv[(size_t)col * N + c];
      }
    }
  }
  return true;
}

// Cyclic Jacobi eigenvalues of a symmetric matrix (for the 2-norm condition number).
std::vector<double> sym_eigvals(std::vector<double> a, int N) {
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int p = 0; p < N; ++p)
      for (int q = 0; q < N; ++q) {
        const double v = a[(size_t)p * N + q] * a[(size_t)p * N + q];
        tot += v;
        if (p != q) off += v;
      }
    if (off <= 1e-30 * tot) break;
    for (int p = 0; p < N - 1; ++p)
      for (int q = p + 1; q < N; ++q) {
        const double apq = a[(size_t)p * N + q];
        if (apq == 0.0) continue;
        const double app = a[(size_t)p * N + p], aqq = a[(size_t)q * N + q];
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) / (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < N; ++k) {
          const double akp = a[(size_t)k * N + p], akq = a[(size_t)k * N + q];
          a[(size_t)k * N + p] = c * akp - s * akq;
          a[(size_t)k * N + q] = s * akp + c * akq;
        }
        for (int k = 0; k < N; ++k) {
          const double apk = a[(size_t)p * N + k], aqk = a[(size_t)q * N + k];
          a[(size_t)p * N + k] = c * apk - s * aqk;
          a[(size_t)q * N + k] = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(N);
  for (int i = 0; i < N; ++i) ev[i] = a[(size_t)i * N + i];
  return ev;
}

// ---------------------------------------------------------------- kernel dispatch
using KernelFn = void (*)(const KParams);

template <int ND, int NXI>
KernelFn pick_big(bool big) {
  return big ? (KernelFn)sf_solve_kernel<ND, NXI, true> : (KernelFn)sf_solve_kernel<ND, NXI, false>;
}

template <int ND>
KernelFn pick_nxi(int nxi, bool big) {
  switch (nxi) {
    case 4: return pick_big<ND, 4>(big);
    case 5: return pick_big<ND, 5>(big);
    case 6: return pick_big<ND, 6>(big);
    case 7: return pick_big<ND, 7>(big);
    case 8: return pick_big<ND, 8>(big);
    case 9: return pick_big<ND, 9>(big);
    case 10: return pick_big<ND, 10>(big);
    case 11: return pick_big<ND, 11>(big);
    case 12: return pick_big<ND, 12>(big);
    default: return nullptr;
  }
}

KernelFn pick_kernel(int nd, int nxi, bool big) {
  return nd == 2 ? pick_nxi<2>(nxi, big) : (nd == 3 ? pick_nxi<3>(nxi, big) : nullptr);
}

int align32(int x) { return (x + 31) & ~31; }

}  // namespace

struct sfb_plan {
  sfb_dims d;
  double rho;
  int mode;
  double cond;
  int device;
  double* d_consts;
  int n_consts;
  Layout L;
  int NKG, LW, RB;
  bool big;
  float plim_base;   // multiplied by the smallest contact axis at solve time
  KernelFn kernel;
};

static bool make_layout(const sfb_dims& d, bool big, Layout& L, int NKG) {
  const int n = d.n, m = d.n_obs, NXI = d.n_basis, NB = d.n_bnd, ND = d.n_d;
  const int ND2 = ND == 2 ? 4 : 8;
  const int nv = ND * n * NXI;
  int off = 0;
  auto take = [&](int bytes) { const int o = off; off = align32(off + bytes); return o; };
  L.xi = take(nv * 8);
  L.lam = take(nv * 8);
  L.w = take(NKG * NXI * 2 * 8);
  L.e = take(NB * NXI * 8);
  L.q = take(NXI * NXI * 8);
  L.pxx = take(NXI * NXI * 8);
  L.pxb = take(NXI * NB * 8);
  L.dxx = take(NXI * NXI * 8);
  L.dxb = take(NXI * NB * 8);
  L.g = take(nv * 8);
  L.bv = take(ND * n * NB * 8);
  L.red = take(NW * 4 * 8 + 32);
  L.obs_ax = take(std::max(m, 1) * 4 * 8);
  L.obs_thr = take(std::max(m, 1) * 2 * 4);
  L.obs = take(std::max(NKG * m * ND2 * 4, 16));
  L.pmax = take(big ? NKG * 8 * 4 : 16);
  const int pos = NKG * n * ND2 * 4 * (big ? 2 : 1);
  const int slot = ND * 32 * NXI * 8;
  const int kkt = (nv + ND * n * NB + ND * NXI + ND * NB) * 8;
  int uni = std::max(pos, std::max(slot, kkt));
  L.uni = take(uni);
  L.uni_bytes = uni;
  L.slots = std::max(1, std::min(NW, uni / slot));
  L.total = off;
  return L.total <= 227 * 1024;
}

extern "C" {

int32_t sfb_abi_version(void) { return SFB_ABI_VERSION; }

const char* sfb_last_error(void) { return g_last_error.c_str(); }

int sfb_plan_create(sfb_plan** out, const sfb_dims* dims, const double* W, const double* Wdd,
                    const double* E, double rho, int32_t mode) {
  if (!out || !dims || !W || !E) return fail(SFB_EINVAL, "null argument");
  *out = nullptr;
  const sfb_dims d = *dims;
  if (d.n < 1 || d.n > 256) return fail(SFB_EINVAL, "n must be in [1, 256]");
  if (d.n_d != 2 && d.n_d != 3) return fail(SFB_EINVAL, "n_d must be 2 or 3");
  if (d.num_steps < 2 || d.n_obs < 0 || d.n_bnd < 1 || d.n_bnd > d.n_basis)
    return fail(SFB_EINVAL, "bad num_steps / n_obs / n_bnd");
  if (!(rho > 0.0)) return fail(SFB_ESETUP, "rho must be positive");
  if (mode != SFB_MODE_PROJECTION && mode != SFB_MODE_SMOOTHNESS)
    return fail(SFB_EINVAL, "unknown objective mode");
  if (mode == SFB_MODE_SMOOTHNESS && !Wdd) return fail(SFB_EINVAL, "smoothness mode needs Wdd");
  const int NXI = d.n_basis, NB = d.n_bnd, K1 = d.num_steps, n = d.n, m = d.n_obs;
  const bool big = n > 32;
  KernelFn kfn = pick_kernel(d.n_d, NXI, big);
  if (!kfn) return fail(SFB_EINVAL, "n_basis must be in [4, 12] for the compiled kernels");

  // S = W^T W, Qb
  std::vector<double> S((size_t)NXI * NXI, 0.0), Qb((size_t)NXI * NXI, 0.0);
  for (int a = 0; a < NXI; ++a)
    for (int c = 0; c < NXI; ++c) {
      double s = 0.0, q = 0.0;
      for (int k = 0; k < K1; ++k) {
        s += W[(size_t)k * NXI + a] * W[(size_t)k * NXI + c];
        if (mode == SFB_MODE_SMOOTHNESS) q += Wdd[(size_t)k * NXI + a] * Wdd[(size_t)k * NXI + c];
      }
      S[(size_t)a * NXI + c] = s;
      Qb[(size_t)a * NXI + c] = (mode == SFB_MODE_PROJECTION) ? (a == c ? 1.0 : 0.0) : q;
    }
  const int NK = NXI + NB;
  auto kkt_block = [&](double cmul) {
    std::vector<double> K((size_t)NK * NK, 0.0);
    for (int a = 0; a < NXI; ++a)
      for (int c = 0; c < NXI; ++c)
        K[(size_t)a * NK + c] = Qb[(size_t)a * NXI + c] + rho * cmul * S[(size_t)a * NXI + c];
    for (int r = 0; r < NB; ++r)
      for (int c = 0; c < NXI; ++c) {
        K[(size_t)c * NK + NXI + r] = E[(size_t)r * NXI + c];
        K[(size_t)(NXI + r) * NK + c] = E[(size_t)r * NXI + c];
      }
    return K;
  };
  // H = I (x) Qb + rho((n+m+2) I - 11^T) (x) S: mean mode K(m+2), n-1 deviation modes K(n+m+2)
  const std::vector<double> Km = kkt_block((double)(m + 2));
  const std::vector<double> Kd = kkt_block((double)(n + m + 2));
  std::vector<double> ev = sym_eigvals(Km, NK);
  if (n > 1) {
    std::vector<double> ev2 = sym_eigvals(Kd, NK);
    ev.insert(ev.end(), ev2.begin(), ev2.end());
  }
  double emax = 0.0, emin = INFINITY;
  for (double v : ev) {
    emax = std::max(emax, std::fabs(v));
    emin = std::min(emin, std::fabs(v));
  }
  const double cond = (emin > 0.0) ? emax / emin : INFINITY;
  if (!(cond <= 1e14)) return fail(SFB_ESETUP, "KKT matrix is singular or near-singular");
  std::vector<double> R, Pm;
  if (!invert(Km, NK, R)) return fail(SFB_ESETUP, "KKT matrix is singular");
  if (n > 1) {
    if (!invert(Kd, NK, Pm)) return fail(SFB_ESETUP, "KKT matrix is singular");
  } else {
    Pm = R;
  }

  const ConstOff co = ConstOff::make(K1, NXI, NB);
  std::vector<double> h((size_t)co.total, 0.0);
  std::memcpy(h.data() + co.W, W, sizeof(double) * K1 * NXI);
  std::memcpy(h.data() + co.E, E, sizeof(double) * NB * NXI);
  std::memcpy(h.data() + co.Q, Qb.data(), sizeof(double) * NXI * NXI);
  const double inv_n = 1.0 / n;
  for (int a = 0; a < NXI; ++a) {
    for (int c = 0; c < NXI; ++c) {
      const double p = Pm[(size_t)a * NK + c], r = R[(size_t)a * NK + c];
      h[co.Pxx + a * NXI + c] = p;
      h[co.Dxx + a * NXI + c] = (r - p) * inv_n;
    }
    for (int rr = 0; rr < NB; ++rr) {
      const double p = Pm[(size_t)a * NK + NXI + rr], r = R[(size_t)a * NK + NXI + rr];
      h[co.Pxb + a * NB + rr] = p;
      h[co.Dxb + a * NB + rr] = (r - p) * inv_n;
    }
  }

  sfb_plan* plan = new sfb_plan();
  plan->d = d;
  plan->rho = rho;
  plan->mode = mode;
  plan->cond = cond;
  plan->kernel = kfn;
  plan->big = big;
  plan->NKG = (K1 + 1) / 2;
  int lw = 1;
  while (lw < n && lw < 32) lw <<= 1;
  plan->LW = lw;
  int rb = (n + 31) / 32;
  int rbp = 1;
  while (rbp < rb) rbp <<= 1;
  plan->RB = rbp;
  // FP32 screen valid while 4 sqrt(n_d) 2^-24 (2P + a) <= ~1e-3 a
  plan->plim_base = (float)(2e-4 / (4.0 * std::sqrt((double)d.n_d) * 5.9604644775390625e-08));
  if (!make_layout(d, big, plan->L, plan->NKG)) {
    delete plan;
    return fail(SFB_EINVAL, "problem too large for one CTA's shared memory");
  }
  cudaError_t e = cudaGetDevice(&plan->device);
  if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaGetDevice"); }
  e = cudaMalloc(&plan->d_consts, sizeof(double) * h.size());
  if (e != cudaSuccess) { delete plan; return cuda_fail(e, "cudaMalloc(plan)"); }
  e = cudaMemcpy(plan->d_consts, h.data(), sizeof(double) * h.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { cudaFree(plan->d_consts); delete plan; return cuda_fail(e, "cudaMemcpy(plan)"); }
  plan->n_consts = (int)h.size();
  e = cudaFuncSetAttribute((const void*)kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, plan->L.total);
  if (e != cudaSuccess) { cudaFree(plan->d_consts); delete plan; return cuda_fail(e, "cudaFuncSetAttribute"); }
  *out = plan;
  return SFB_OK;
}

void sfb_plan_destroy(sfb_plan* plan) {
  if (!plan) return;
  if (plan->d_consts) cudaFree(plan->d_consts);
  delete plan;
}

double sfb_plan_cond(const sfb_plan* plan) { return plan ? plan->cond : NAN; }

int64_t sfb_smem_bytes(const sfb_plan* plan) { return plan ? plan->L.total : 0; }

int sfb_solve(const sfb_plan* plan, const sfb_batch* bt, const sfb_config* cfg,
              const sfb_out* out, void* stream) {
  if (!plan || !bt || !cfg || !out) return fail(SFB_EINVAL, "null argument");
  if (bt->n_members < 0 || bt->n_instances < 1) return fail(SFB_EINVAL, "bad batch size");
  if (bt->n_members == 0) return SFB_OK;
  if (!bt->member_instance || !bt->xi0 || !bt->lam0 || !bt->bvals || !bt->box || !bt->pair_axes)
    return fail(SFB_EINVAL, "missing batch buffer");
  if (plan->d.n_obs > 0 && (!bt->obs_pos || !bt->obs_axes)) return fail(SFB_EINVAL, "missing obstacle buffers");
  if (plan->mode == SFB_MODE_PROJECTION && !bt->target) return fail(SFB_EINVAL, "projection mode needs a target");
  if (!out->xi || !out->lam || !out->primal || !out->eq_max || !out->iterations || !out->status)
    return fail(SFB_EINVAL, "missing output buffer");
  if (cfg->rho != plan->rho) return fail(SFB_EINVAL, "cfg.rho differs from the plan's rho");
  if (cfg->max_iters < 0) return fail(SFB_EINVAL, "max_iters must be >= 0");
  if (!(cfg->primal_tol > 0.0 && cfg->fp_tol > 0.0)) return fail(SFB_ESETUP, "tolerances must be positive");
  int dev = -1;
  cudaGetDevice(&dev);
  if (dev != plan->device) return fail(SFB_EINVAL, "plan was created on another device");

  KParams P;
  std::memset(&P, 0, sizeof(P));
  const sfb_dims& d = plan->d;
  P.n = d.n; P.m = d.n_obs; P.K1 = d.num_steps; P.NB = d.n_bnd; P.NKG = plan->NKG;
  P.LW = plan->LW; P.RB = plan->RB;
  P.mode = plan->mode; P.max_iters = cfg->max_iters; P.early_exit = cfg->early_exit ? 1 : 0;
  P.rho = cfg->rho; P.primal_tol = cfg->primal_tol; P.fp_tol = cfg->fp_tol; P.d_max = cfg->d_max;
  P.inv_n = 1.0 / d.n;
  P.L = plan->L;
  P.consts = plan->d_consts;
  P.B = bt->n_members;
  P.member_instance = bt->member_instance;
  P.xi0 = bt->xi0; P.lam0 = bt->lam0; P.target = plan->mode == SFB_MODE_PROJECTION ? bt->target : nullptr;
  P.bvals = bt->bvals; P.box = bt->box; P.obs_pos = bt->obs_pos; P.obs_axes = bt->obs_axes;
  P.pair_axes = bt->pair_axes;
  P.xi = out->xi; P.lam = out->lam; P.primal = out->primal; P.eq_max = out->eq_max;
  P.iterations = out->iterations; P.status = out->status; P.trace = out->trace;
  P.counters = reinterpret_cast<unsigned long long*>(out->counters);
  P.plim = plan->plim_base;  // scaled in-kernel by the member's smallest contact axis
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  (void)cudaGetLastError();  // do not report a stale error of an unrelated earlier call
  if (out->counters) {
    cudaError_t e = cudaMemsetAsync(out->counters, 0, sizeof(uint64_t) * 4 * (size_t)bt->n_members, s);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(counters)");
  }
  // the attribute is per kernel instance, shared by plans of different shapes
  cudaError_t e = cudaFuncSetAttribute((const void*)plan->kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, plan->L.total);
  if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute");
  plan->kernel<<<bt->n_members, NT, plan->L.total, s>>>(P);
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[160];
    std::snprintf(buf, sizeof(buf), "sf_solve_kernel launch (B=%d, smem=%d)", bt->n_members, plan->L.total);
    return cuda_fail(e, buf);
  }
  return SFB_OK;
}

}  // extern "C"
