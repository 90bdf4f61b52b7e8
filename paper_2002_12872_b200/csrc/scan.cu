// scan.cu -- batched scan_domain (proj/src/analysis.cpp:68-138): every cell of
// a lambda grid is one small DPT solve; here one WARP solves one cell with the
// whole state machine on chip, and the grid of warps covers all cells in one
// launch (the reference spawns a thread pool and solves cell after cell).
//
// Arithmetic follows the reference operation by operation, so classes and
// iteration counts match it: complex products are (ac - bd, ad + bc) with every
// product and sum rounded separately (no FMA contraction -- the reference's
// x86-64 build has none), matmul accumulates in k order and skips a(i,k) == 0
// (proj/src/matrix.cpp:130-143), matvec accumulates in j order (:215-225),
// magnitudes are hypot (std::abs of a complex), theta and the gap row are the
// host's std::complex divisions (proj/src/partition.cpp:69-96) uploaded as
// tables, and the ramp factors 1 - alpha^(k-1) are the host's std::pow.
//
// Full mode restates run_full (proj/src/dpt.cpp:92-192); row mode restates
// run_single (:194-293).  A cell's iterates live in shared memory
// (4 n^2 complex per warp, n <= NMAX); the cycle window's past iterates live
// in a per-warp global ring (L2).
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_kernels.h"

namespace dpt {

namespace {

struct C {
  double x, y;
};
__device__ __forceinline__ C mk(double x, double y) { return C{x, y}; }
__device__ __forceinline__ C add(C a, C b) { return C{__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y)}; }
__device__ __forceinline__ C sub(C a, C b) { return C{__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y)}; }
__device__ __forceinline__ C mul(C a, C b) {
  return C{__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x))};
}
__device__ __forceinline__ double cabs(C a) { return hypot(a.x, a.y); }
__device__ __forceinline__ bool finite(C a) { return isfinite(a.x) && isfinite(a.y); }
__device__ __forceinline__ C ld(const double* p, int64_t i) { return C{__ldg(p + 2 * i), __ldg(p + 2 * i + 1)}; }

__device__ __forceinline__ double wmax(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

constexpr int kWarpsMax = 16;

// status codes as ConvergenceStatus; classify() maps MaxIterations to Bounded.
__device__ __forceinline__ uint8_t cell_class(int status) { return status == 0 ? 0 : (status == 2 ? 2 : 1); }

// Shared-memory layout of a block: [tables][warp 0 area][warp 1 area]...;
// the read-only tables (full: Delta^T, theta; row: Delta, gap row) are staged
// once per block so every complex MAC reads shared memory, not L1.
__device__ __forceinline__ void stage(C* dst, const double* src, int count) {
  for (int q = threadIdx.x; q < count; q += blockDim.x) dst[q] = C{src[2 * q], src[2 * q + 1]};
}

template <int NMAX>
__global__ void __launch_bounds__(32 * kWarpsMax) scan_full_kernel(ScanArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = a.n, nn = n * n;
  C* const DT = reinterpret_cast<C*>(smem);  // Delta^T
  C* const TH = DT + NMAX * NMAX;             // theta
  stage(DT, a.delta_t, nn);
  stage(TH, a.theta, nn);
  __syncthreads();
  C* A = TH + NMAX * NMAX + size_t(wib) * size_t(a.warp_elems);
  C* An = A + NMAX * NMAX;
  C* P = An + NMAX * NMAX;
  C* Pn = P + NMAX * NMAX;
  const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int win = a.win;  // effective_window (host)
  const int nring = win > 1 ? win - 1 : 0;
  C* ring = a.ring_smem ? Pn + NMAX * NMAX  // after this warp's four matrices
                        : reinterpret_cast<C*>(a.ring) + size_t(gw) * size_t(nring) * size_t(nn);
  const int rstride = a.ring_smem ? NMAX * NMAX : nn;
  const double tol = a.tol, margin = 1e3 * a.tol;
  for (int64_t cell = gw; cell < a.cells; cell += nw) {
    const int64_t ii = cell / a.res_re, jj = cell % a.res_re;
    const C lam = mk(a.re_at[jj], a.im_at[ii]);
    const double lam_abs = cabs(lam);
    // A = I, P = A * delta_t = delta_t (skip of zero a(i,k): row i of P is row i of delta_t)
    for (int e = lane; e < nn; e += 32) {
      const int i = e / n, j = e % n;
      A[e] = mk(i == j ? 1.0 : 0.0, 0.0);
      P[e] = add(mk(0.0, 0.0), mul(mk(1.0, 0.0), DT[i * n + j]));
    }
    __syncwarp();
    int status = 3, iters = a.max_iter, filled = 0, head = 0;
    for (int k = 1; k <= a.max_iter; ++k) {
      const C lam_k = a.ramp ? C{__dmul_rn(lam.x, a.ramp[k]), __dmul_rn(lam.y, a.ramp[k])} : lam;
      const bool settled = !a.ramp || cabs(sub(lam_k, lam)) <= __dmul_rn(tol, lam_abs);
      double step = 0.0, mabs = 0.0;
      bool fin = true;
      for (int e = lane; e < nn; e += 32) {
        const int i = e / n, j = e % n;
        C v;
        if (i == j) {
          v = mk(1.0, 0.0);
        } else {
          v = mul(mul(lam_k, TH[e]), sub(P[e], mul(P[i * n + i], A[e])));
        }
        An[e] = v;
        step = fmax(step, cabs(sub(v, A[e])));
        mabs = fmax(mabs, cabs(v));
        fin = fin && finite(v);
      }
      step = wmax(step);
      mabs = wmax(mabs);
      fin = __all_sync(0xffffffffu, fin);
      if (!fin || mabs > a.div_thr) {
        status = 2;
        iters = k;
        break;
      }
      __syncwarp();
      // Pn = An * delta_t, k order, zero a(i,k) skipped (matrix.cpp:130-143).
      // A lane's entries advance together, TB at a time, one k per step: TB
      // independent dependency chains in flight instead of one (each entry
      // still sums its terms in k order, so the result is unchanged).
      {
        constexpr int T = (NMAX * NMAX + 31) / 32, TB = T < 8 ? T : 8;
        for (int t0 = 0; t0 < T; t0 += TB) {
          C acc[TB];
          int ei[TB], ej[TB];
#pragma unroll
          for (int u = 0; u < TB; ++u) {
            const int e = lane + 32 * (t0 + u);
            const int ee = e < nn ? e : 0;
            ei[u] = ee / n;
            ej[u] = ee % n;
            acc[u] = mk(0.0, 0.0);
          }
          for (int q = 0; q < n; ++q) {
#pragma unroll
            for (int u = 0; u < TB; ++u) {
              const C aik = An[ei[u] * n + q];
              if (!(aik.x == 0.0 && aik.y == 0.0)) acc[u] = add(acc[u], mul(aik, DT[q * n + ej[u]]));
            }
          }
#pragma unroll
          for (int u = 0; u < TB; ++u) {
            const int e = lane + 32 * (t0 + u);
            if (e < nn) Pn[e] = acc[u];
          }
        }
      }
      __syncwarp();
      bool stop = false;
      if (settled && step < tol) {
        // residuals_of (dpt.cpp:23-44): lane i owns row i
        double worst = 0.0;
        for (int i = lane; i < n; i += 32) {
          const C eps = add(ld(a.d, i), mul(lam, Pn[i * n + i]));
          double num = 0.0, den = 0.0;
          for (int m = 0; m < n; ++m) {
            const C r = add(mul(sub(ld(a.d, m), eps), An[i * n + m]), mul(lam, Pn[i * n + m]));
            num = fmax(num, cabs(r));
            den = fmax(den, cabs(An[i * n + m]));
          }
          worst = fmax(worst, num / fmax(den, 1e-300));
        }
        worst = wmax(worst);
        if (worst < a.res_tol) {
          status = 0;
          iters = k;
          stop = true;
        }
      } else if (win > 0 && settled && step > margin && filled > 0) {
        // within_tol against every window entry at once: bit s of `differs`
        // = "ring slot s has a component >= tol away"; Bounded if any filled
        // slot has none (which one is irrelevant to the outcome)
        // Sample first: entry `lane` of every slot (one load per slot per
        // lane) refutes almost every slot; only the survivors are compared
        // in full.  Exact: a refuted slot has a component >= tol away.
        bool within_any = false;
        const C cv0 = lane < nn ? An[lane] : mk(0.0, 0.0);
        for (int s0 = 0; s0 < filled && !within_any; s0 += 32) {  // 32 slots per mask
          const int cnt = filled - s0 < 32 ? filled - s0 : 32;
          unsigned differs = 0u;
          if (lane < nn)
            for (int sl = 0; sl < cnt; ++sl) {
              const C pv = ring[size_t(s0 + sl) * size_t(rstride) + lane];
              if (fabs(__dsub_rn(cv0.x, pv.x)) >= tol || fabs(__dsub_rn(cv0.y, pv.y)) >= tol) differs |= 1u << sl;
            }
          differs = __reduce_or_sync(0xffffffffu, differs);
          const unsigned full_mask = cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u);
          unsigned open = full_mask & ~differs;  // slots the sample did not refute
          while (open && !within_any) {
            const int sl = __ffs(open) - 1;
            open &= open - 1;
            bool d = false;
            for (int e = lane + 32; e < nn; e += 32) {
              const C pv = ring[size_t(s0 + sl) * size_t(rstride) + e], cv = An[e];
              if (fabs(__dsub_rn(cv.x, pv.x)) >= tol || fabs(__dsub_rn(cv.y, pv.y)) >= tol) d = true;
            }
            within_any = !__any_sync(0xffffffffu, d);
          }
        }
        if (within_any) {
          status = 1;
          iters = k;
          stop = true;
        }
      }
      if (stop) break;
      if (nring > 0) {  // window.push_front(a), at most win - 1 entries (slot order is irrelevant)
        C* dst = ring + size_t(head) * size_t(rstride);
        for (int e = lane; e < nn; e += 32) dst[e] = A[e];
        head = (head + 1) % nring;
        if (filled < nring) ++filled;
      }
      for (int e = lane; e < nn; e += 32) {
        A[e] = An[e];
        P[e] = Pn[e];
      }
      __syncwarp();
    }
    if (lane == 0) {
      a.classes[cell] = cell_class(status);
      a.iterations[cell] = iters;
    }
    __syncwarp();
  }
}

template <int NMAX, bool STAGE>
__global__ void __launch_bounds__(32 * kWarpsMax) scan_single_kernel(ScanArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n = a.n;
  C* const DL = reinterpret_cast<C*>(smem);     // Delta (STAGE)
  C* const GR = DL + (STAGE ? NMAX * NMAX : 0);  // gap row (STAGE)
  if (STAGE) {
    stage(DL, a.delta, n * n);
    stage(GR, a.gap_row, n);
    __syncthreads();
  }
  auto dl = [&](int m, int q) -> C { return STAGE ? DL[m * n + q] : ld(a.delta, int64_t(m) * n + q); };
  auto gr = [&](int m) -> C { return STAGE ? GR[m] : ld(a.gap_row, m); };
  C* z = GR + (STAGE ? NMAX : 0) + size_t(wib) * size_t(a.warp_elems);
  C* zn = z + NMAX;
  C* w = zn + NMAX;
  C* wn = w + NMAX;
  const int64_t gw = int64_t(blockIdx.x) * (blockDim.x >> 5) + wib;
  const int64_t nw = int64_t(gridDim.x) * (blockDim.x >> 5);
  const int win = a.win;  // cycle_window if >= 2 (no cap, dpt.cpp:207)
  const int nring = win > 1 ? win - 1 : 0;
  C* ring = a.ring_smem ? wn + NMAX : reinterpret_cast<C*>(a.ring) + size_t(gw) * size_t(nring) * size_t(n);
  const int rstride = a.ring_smem ? NMAX : n;
  const double tol = a.tol, margin = 1e3 * a.tol;
  const int row = a.row;
  for (int64_t cell = gw; cell < a.cells; cell += nw) {
    const int64_t ii = cell / a.res_re, jj = cell % a.res_re;
    const C lam = mk(a.re_at[jj], a.im_at[ii]);
    const double lam_abs = cabs(lam);
    for (int m = lane; m < n; m += 32) z[m] = mk(m == row ? 1.0 : 0.0, 0.0);
    __syncwarp();
    for (int m = lane; m < n; m += 32) {  // w = matvec(delta, z), j order
      C s = mk(0.0, 0.0);
      for (int q = 0; q < n; ++q) s = add(s, mul(dl(m, q), z[q]));
      w[m] = s;
    }
    __syncwarp();
    int status = 3, iters = a.max_iter, filled = 0, head = 0;
    for (int k = 1; k <= a.max_iter; ++k) {
      const C lam_k = a.ramp ? C{__dmul_rn(lam.x, a.ramp[k]), __dmul_rn(lam.y, a.ramp[k])} : lam;
      const bool settled = !a.ramp || cabs(sub(lam_k, lam)) <= __dmul_rn(tol, lam_abs);
      const C wrow = w[row];
      double step = 0.0, mabs = 0.0;
      bool fin = true;
      for (int m = lane; m < n; m += 32) {
        const C v = m == row ? mk(1.0, 0.0) : mul(mul(lam_k, gr(m)), sub(w[m], mul(wrow, z[m])));
        zn[m] = v;
        step = fmax(step, cabs(sub(v, z[m])));
        mabs = fmax(mabs, cabs(v));
        fin = fin && finite(v);
      }
      step = wmax(step);
      mabs = wmax(mabs);
      fin = __all_sync(0xffffffffu, fin);
      if (!fin || mabs > a.div_thr) {
        status = 2;
        iters = k;
        break;
      }
      __syncwarp();
      for (int m = lane; m < n; m += 32) {
        C s = mk(0.0, 0.0);
        for (int q = 0; q < n; ++q) s = add(s, mul(dl(m, q), zn[q]));
        wn[m] = s;
      }
      __syncwarp();
      bool stop = false;
      if (settled && step < tol) {
        // residual_single (dpt.cpp:47-58) with eps = d_row + lam wnext[row]
        const C eps = add(ld(a.d, row), mul(lam, wn[row]));
        double num = 0.0, den = 0.0;
        for (int m = lane; m < n; m += 32) {
          const C r = add(mul(sub(ld(a.d, m), eps), zn[m]), mul(lam, wn[m]));
          num = fmax(num, cabs(r));
          den = fmax(den, cabs(zn[m]));
        }
        num = wmax(num);
        den = wmax(den);
        if (num / fmax(den, 1e-300) < a.res_tol) {
          status = 0;
          iters = k;
          stop = true;
        }
      } else if (win > 0 && settled && step > margin && filled > 0) {
        // all window entries at once (see the full kernel); the ring holds at
        // most 31 entries per pass of the mask, more are checked in rounds
        bool within_any = false;  // sample first (see the full kernel), then the survivors in full
        const C cv0 = lane < n ? zn[lane] : mk(0.0, 0.0);
        for (int s0 = 0; s0 < filled && !within_any; s0 += 32) {
          const int cnt = filled - s0 < 32 ? filled - s0 : 32;
          unsigned differs = 0u;
          if (lane < n)
            for (int sl = 0; sl < cnt; ++sl) {
              const C pv = ring[size_t(s0 + sl) * size_t(rstride) + lane];
              if (fabs(__dsub_rn(cv0.x, pv.x)) >= tol || fabs(__dsub_rn(cv0.y, pv.y)) >= tol) differs |= 1u << sl;
            }
          differs = __reduce_or_sync(0xffffffffu, differs);
          const unsigned full_mask = cnt == 32 ? 0xffffffffu : ((1u << cnt) - 1u);
          unsigned open = full_mask & ~differs;
          while (open && !within_any) {
            const int sl = __ffs(open) - 1;
            open &= open - 1;
            bool d = false;
            for (int m = lane + 32; m < n; m += 32) {
              const C pv = ring[size_t(s0 + sl) * size_t(rstride) + m], cv = zn[m];
              if (fabs(__dsub_rn(cv.x, pv.x)) >= tol || fabs(__dsub_rn(cv.y, pv.y)) >= tol) d = true;
            }
            within_any = !__any_sync(0xffffffffu, d);
          }
        }
        if (within_any) {
          status = 1;
          iters = k;
          stop = true;
        }
      }
      if (stop) break;
      if (nring > 0) {
        C* dst = ring + size_t(head) * size_t(rstride);
        for (int m = lane; m < n; m += 32) dst[m] = z[m];
        head = (head + 1) % nring;
        if (filled < nring) ++filled;
      }
      for (int m = lane; m < n; m += 32) {
        z[m] = zn[m];
        w[m] = wn[m];
      }
      __syncwarp();
    }
    if (lane == 0) {
      a.classes[cell] = cell_class(status);
      a.iterations[cell] = iters;
    }
    __syncwarp();
  }
}

// ---- tiny problems (n <= 3, the reference's 2x2 / 3x3 fixtures): one THREAD
// per cell, iterates in registers.  Each lane runs its own cell's state
// machine one iteration per trip and starts its next cell as soon as the
// current one terminates, so lanes stay busy although cells need different
// iteration counts.  Same operation order as the warp kernels.  The window
// ring is per thread in global memory, [slot][entry][thread] (coalesced).
template <int N, bool SINGLE>
__global__ void __launch_bounds__(128) scan_tiny_kernel(ScanArgs a) {
  constexpr int NN = SINGLE ? N : N * N;
  __shared__ C DT[N * N];  // full: Delta^T; row: Delta
  __shared__ C TH[N * N];  // full: theta; row: gap row (first N)
  __shared__ C DL[N];
  for (int q = threadIdx.x; q < N * N; q += blockDim.x) {
    DT[q] = ld(SINGLE ? a.delta : a.delta_t, q);
    TH[q] = (SINGLE ? q < N : true) ? ld(SINGLE ? a.gap_row : a.theta, q) : mk(0.0, 0.0);
  }
  for (int q = threadIdx.x; q < N; q += blockDim.x) DL[q] = ld(a.d, q);
  __syncthreads();
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nthreads = int64_t(gridDim.x) * blockDim.x;
  const int win = a.win, nring = win > 1 ? win - 1 : 0;
  const double tol = a.tol, margin = 1e3 * a.tol;
  const int row = a.row;
  C A[NN], P[NN];  // full: A, P = A Delta^T; row: z, w = Delta z
  C lam = mk(0.0, 0.0);
  double lam_abs = 0.0;
  int k = 1, filled = 0, head = 0;
  int64_t cell = tid;
  auto ring = [&](int slot, int e) -> C& {
    return reinterpret_cast<C*>(a.ring)[(size_t(slot) * NN + e) * size_t(nthreads) + size_t(tid)];
  };
  auto start = [&]() {
    const int64_t ii = cell / a.res_re, jj = cell % a.res_re;
    lam = mk(a.re_at[jj], a.im_at[ii]);
    lam_abs = cabs(lam);
    k = 1;
    filled = 0;
    head = 0;
    if (SINGLE) {
#pragma unroll
      for (int m = 0; m < N; ++m) A[m] = mk(m == row ? 1.0 : 0.0, 0.0);
#pragma unroll
      for (int m = 0; m < N; ++m) {
        C s2 = mk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < N; ++q) s2 = add(s2, mul(DT[m * N + q], A[q]));
        P[m] = s2;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NN; ++e) {
        A[e] = mk(e / N == e % N ? 1.0 : 0.0, 0.0);
        P[e] = add(mk(0.0, 0.0), mul(mk(1.0, 0.0), DT[e]));
      }
    }
  };
  auto finish = [&](int status, int iters) {
    a.classes[cell] = cell_class(status);
    a.iterations[cell] = iters;
    cell += nthreads;
  };
  bool active = cell < a.cells;
  if (active) start();
  while (__any_sync(0xffffffffu, active)) {
    if (!active) continue;
    if (k > a.max_iter) {  // MaxIterations (also max_iter <= 0)
      finish(3, a.max_iter);
      active = cell < a.cells;
      if (active) start();
      continue;
    }
    const C lam_k = a.ramp ? C{__dmul_rn(lam.x, a.ramp[k]), __dmul_rn(lam.y, a.ramp[k])} : lam;
    const bool settled = !a.ramp || cabs(sub(lam_k, lam)) <= __dmul_rn(tol, lam_abs);
    C An[NN], Pn[NN];
    double step = 0.0, mabs = 0.0;
    bool fin = true;
    if (SINGLE) {
      C wrow = mk(0.0, 0.0);  // P[row] without a dynamic register index
#pragma unroll
      for (int m = 0; m < N; ++m)
        if (m == row) wrow = P[m];
#pragma unroll
      for (int m = 0; m < N; ++m) {
        An[m] = m == row ? mk(1.0, 0.0) : mul(mul(lam_k, TH[m]), sub(P[m], mul(wrow, A[m])));
        step = fmax(step, cabs(sub(An[m], A[m])));
        mabs = fmax(mabs, cabs(An[m]));
        fin = fin && finite(An[m]);
      }
    } else {
#pragma unroll
      for (int e = 0; e < NN; ++e) {
        const int i = e / N;
        An[e] = (i == e % N) ? mk(1.0, 0.0) : mul(mul(lam_k, TH[e]), sub(P[e], mul(P[i * N + i], A[e])));
        step = fmax(step, cabs(sub(An[e], A[e])));
        mabs = fmax(mabs, cabs(An[e]));
        fin = fin && finite(An[e]);
      }
    }
    if (!fin || mabs > a.div_thr) {
      finish(2, k);
      active = cell < a.cells;
      if (active) start();
      continue;
    }
    if (SINGLE) {
#pragma unroll
      for (int m = 0; m < N; ++m) {
        C s2 = mk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < N; ++q) s2 = add(s2, mul(DT[m * N + q], An[q]));
        Pn[m] = s2;
      }
    } else {
#pragma unroll
      for (int e = 0; e < NN; ++e) {
        const int i = e / N, j = e % N;
        C s2 = mk(0.0, 0.0);
#pragma unroll
        for (int q = 0; q < N; ++q) {
          const C aik = An[i * N + q];
          if (aik.x == 0.0 && aik.y == 0.0) continue;
          s2 = add(s2, mul(aik, DT[q * N + j]));
        }
        Pn[e] = s2;
      }
    }
    int status = -1;
    if (settled && step < tol) {
      double worst = 0.0;
      if (SINGLE) {
        C pr = mk(0.0, 0.0);
#pragma unroll
        for (int m = 0; m < N; ++m)
          if (m == row) pr = Pn[m];
        const C eps = add(DL[row], mul(lam, pr));
        double num = 0.0, den = 0.0;
#pragma unroll
        for (int m = 0; m < N; ++m) {
          num = fmax(num, cabs(add(mul(sub(DL[m], eps), An[m]), mul(lam, Pn[m]))));
          den = fmax(den, cabs(An[m]));
        }
        worst = num / fmax(den, 1e-300);
      } else {
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const C eps = add(DL[i], mul(lam, Pn[i * N + i]));
          double num = 0.0, den = 0.0;
#pragma unroll
          for (int m = 0; m < N; ++m) {
            num = fmax(num, cabs(add(mul(sub(DL[m], eps), An[i * N + m]), mul(lam, Pn[i * N + m]))));
            den = fmax(den, cabs(An[i * N + m]));
          }
          worst = fmax(worst, num / fmax(den, 1e-300));
        }
      }
      if (worst < a.res_tol) status = 0;
    } else if (win > 0 && settled && step > margin) {
      for (int p = 0; p < filled && status < 0; ++p) {
        bool within = true;
#pragma unroll
        for (int e = 0; e < NN; ++e) {
          const C pv = ring(p, e);
          if (fabs(__dsub_rn(An[e].x, pv.x)) >= tol || fabs(__dsub_rn(An[e].y, pv.y)) >= tol) within = false;
        }
        if (within) status = 1;
      }
    }
    if (status >= 0) {
      finish(status, k);
      active = cell < a.cells;
      if (active) start();
      continue;
    }
    if (nring > 0) {
#pragma unroll
      for (int e = 0; e < NN; ++e) ring(head, e) = A[e];
      head = head + 1 == nring ? 0 : head + 1;
      if (filled < nring) ++filled;
    }
#pragma unroll
    for (int e = 0; e < NN; ++e) {
      A[e] = An[e];
      P[e] = Pn[e];
    }
    ++k;
  }
}

template <int NMAX>
cudaError_t launch_scan_t(ScanArgs a, int warps_total, cudaStream_t st) {
  const int unit = a.single ? NMAX : NMAX * NMAX;  // complex elements per vector / matrix
  const int nring = a.win > 1 ? a.win - 1 : 0;
  // the window ring on chip only while it keeps >= 32 warps per SM resident;
  // otherwise in L2 (the all-entries check costs one round trip either way)
  a.ring_smem = (4 + nring) * unit * 16 <= 6 * 1024 ? 1 : 0;
  a.warp_elems = (4 + (a.ring_smem ? nring : 0)) * unit;
  constexpr bool kStageSingle = NMAX <= 64;  // Delta (n^2 complex) fits beside the warp areas
  const size_t tables = a.single ? (kStageSingle ? size_t(NMAX * NMAX + NMAX) * 16 : 0)
                                 : size_t(2 * NMAX * NMAX) * 16;
  const int per_warp = a.warp_elems * 16;
  int wpb = int((200 * 1024 - tables) / size_t(per_warp));
  if (wpb > kWarpsMax) wpb = kWarpsMax;
  if (wpb < 1) wpb = 1;
  const int blocks = (warps_total + wpb - 1) / wpb;
  const size_t smem = tables + size_t(wpb) * size_t(per_warp);
  if (a.single) {
    auto k = scan_single_kernel<NMAX, kStageSingle>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    k<<<blocks, 32 * wpb, smem, st>>>(a);
  } else {
    cudaFuncSetAttribute(scan_full_kernel<NMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    scan_full_kernel<NMAX><<<blocks, 32 * wpb, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace

int scan_max_n(int single) { return single ? 2048 : 32; }

int64_t scan_tiny_threads(const ScanArgs& a) {
  if (a.n > 3) return 0;
  int64_t t = a.cells < 148 * 2048 ? a.cells : 148 * 2048;
  return (t + 127) / 128 * 128;
}

cudaError_t launch_scan(const ScanArgs& a, int warps_total, cudaStream_t st) {
  if (a.n <= 3) {  // thread per cell; the caller sized the ring for scan_tiny_threads(a) threads
    const int64_t t = scan_tiny_threads(a);
    const unsigned blocks = unsigned(t / 128);
#define DPT_TINY(NV)                                                      \
  if (a.n == NV) {                                                        \
    if (a.single)                                                         \
      scan_tiny_kernel<NV, true><<<blocks, 128, 0, st>>>(a);             \
    else                                                                  \
      scan_tiny_kernel<NV, false><<<blocks, 128, 0, st>>>(a);            \
    return cudaGetLastError();                                            \
  }
    DPT_TINY(1)
    DPT_TINY(2)
    DPT_TINY(3)
#undef DPT_TINY
  }
  if (a.single) {
    if (a.n <= 32) return launch_scan_t<32>(a, warps_total, st);
    if (a.n <= 64) return launch_scan_t<64>(a, warps_total, st);
    if (a.n <= 128) return launch_scan_t<128>(a, warps_total, st);
    if (a.n <= 256) return launch_scan_t<256>(a, warps_total, st);
    if (a.n <= 2048) return launch_scan_t<2048>(a, warps_total, st);
    return cudaErrorInvalidValue;
  }
  if (a.n <= 4) return launch_scan_t<4>(a, warps_total, st);
  if (a.n <= 8) return launch_scan_t<8>(a, warps_total, st);
  if (a.n <= 16) return launch_scan_t<16>(a, warps_total, st);
  if (a.n <= 32) return launch_scan_t<32>(a, warps_total, st);
  return cudaErrorInvalidValue;
}

}  // namespace dpt
