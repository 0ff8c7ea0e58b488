// solve.cu — the inner linear solves.
//
// k_schwarz: one sweep of the reference's alternating-Schwarz iteration
// (schwarz_iterate, solver.cpp:414-482): every subdomain (16 px tile of grid
// nodes, build_subdomains solver.cpp:382-412) runs pcg_iters PCG iterations
// (pcg_impl, solver.cpp:320-361) on its interior unknowns, warm-started from the
// published values, with off-subdomain neighbours frozen at the previous
// sweep's published values. One thread per local unknown; a "team" (one warp
// for step >= 8, i.e. <= 24 unknowns) owns one subdomain; the team's rows of
// the local matrix live in registers for the whole sweep; dots are xor-butterfly
// warp sums (deterministic, identical in every lane). The last sweep fuses the
// Gauss-Newton update delta += step, total = base + delta (solver.cpp:518-523).
//
// k_pcg_global: the subdomain_px = 0 mode (pcg_solve, solver.cpp:365-380), one
// CTA per frame pair looping over all iterations with block-wide fixed-order dots.
#include <algorithm>
#include <cstdlib>

#include <cooperative_groups.h>

#include "launch.h"

namespace hwf {
namespace cg = cooperative_groups;
namespace {

// Row r of block(n, slot9) of the symmetric system.
__device__ __forceinline__ double sys_entry(const double* __restrict__ sys, int G, int n, int nb,
                                            int s9, int r, int c) {
  if (s9 >= 4) return __ldg(sys + static_cast<size_t>(n) * kSysStride + (s9 - 4) * 21 + sym6(r, c));
  return __ldg(sys + static_cast<size_t>(nb) * kSysStride + (4 - s9) * 21 + sym6(r, c));
}

template <int TEAM>
__device__ __forceinline__ double team_sum(double v, double* scratch) {
  v = warp_sum(v);
  if (TEAM == 32) return v;
  const int lane = threadIdx.x & 31, wt = (threadIdx.x % TEAM) >> 5;
  __syncthreads();
  if (lane == 0) scratch[wt] = v;
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < TEAM / 32; ++k) s += scratch[k];
  return s;
}

// NLOC > 0: tiles of <= NLOC nodes, one warp per subdomain, each lane keeps
// its dense local row (NLOC nodes x 6) in registers. NLOC == 0: general tiles,
// a team of TEAM threads, 9-slot rows.
template <int TEAM, int NLOC>
__global__ void __launch_bounds__(TEAM == 32 ? 128 : TEAM) k_schwarz(const SwzArgs a) {
  constexpr int SUBS = TEAM == 32 ? 4 : 1;
  constexpr int NR = NLOC > 0 ? NLOC : 9;  // row blocks held per lane
  __shared__ double psh[SUBS][TEAM];
  __shared__ double scratch[TEAM / 32 + 1];
  const int team = threadIdx.x / TEAM, u = threadIdx.x % TEAM;
  const int pair = blockIdx.y;
  const int sub = a.sub0 + blockIdx.x * SUBS + team;
  const int G = a.gw * a.gh;
  const bool sub_ok = sub < a.sub1;
  const int tx = sub_ok ? sub % a.ntx : 0, ty = sub_ok ? sub / a.ntx : 0;
  const int alo = (tx * a.tile + a.step - 1) / a.step, ahi = min(a.gw - 1, ((tx + 1) * a.tile - 1) / a.step);
  const int blo = (ty * a.tile + a.step - 1) / a.step, bhi = min(a.gh - 1, ((ty + 1) * a.tile - 1) / a.step);
  const int i = u / 6, r = u % 6;
  const int ix = i % a.nxm, iy = i / a.nxm;
  const int na = alo + ix, nb = blo + iy;
  const bool act = sub_ok && i < a.nxm * a.nym && na <= ahi && nb <= bhi;
  const int n = act ? nb * a.gw + na : 0;
  const double* sys = a.sys + static_cast<size_t>(pair) * G * kSysStride;
  const double* pub = a.pub ? a.pub + static_cast<size_t>(pair) * G * 6 : nullptr;
  double* psub = psh[team];

  double arow[NR][6];
  int lidx[NR];
  double b = 0.0, x = 0.0;
  // packed offsets of row r in a symmetric 6x6 block: sym6(r, c) for c = 0..5
  int ro[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) ro[c] = sym6(r, c);
  const double* sysn = sys + static_cast<size_t>(n) * kSysStride;
  if (act) {
    b = __ldg(sysn + kSysRhs + r);
    if (pub) x = __ldg(pub + 6 * static_cast<size_t>(n) + r);
  }
  if (NLOC > 0) {
#pragma unroll
    for (int j = 0; j < NR; ++j) {  // dense local row over the tile's nodes
      const int jx = j % a.nxm, jy = j / a.nxm;
      const int qa = alo + jx, qb = blo + jy;
      const bool ok = act && j < a.nxm * a.nym && qa <= ahi && qb <= bhi && abs(qa - na) <= 1 && abs(qb - nb) <= 1;
      const int s9 = (qb - nb + 1) * 3 + (qa - na + 1);
      const double* blk = s9 >= 4 ? sysn + (s9 - 4) * 21 : sys + static_cast<size_t>(qb * a.gw + qa) * kSysStride + (4 - s9) * 21;
      lidx[j] = 6 * j;
#pragma unroll
      for (int c = 0; c < 6; ++c) arow[j][c] = ok ? __ldg(blk + ro[c]) : 0.0;
    }
  }
  if (NLOC > 0 && pub) {
    // coupling to the frozen neighbours (solver.cpp:437-448), two alternating chains
    double b0 = 0.0, b1 = 0.0;
#pragma unroll
    for (int s9 = 0; s9 < 9; ++s9) {
      if (s9 == 4) continue;
      const int qa = na + s9 % 3 - 1, qb = nb + s9 / 3 - 1;
      const bool valid = act && qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh;
      const bool local = qa >= alo && qa <= ahi && qb >= blo && qb <= bhi;
      if (!valid || local) continue;
      const int qn = qb * a.gw + qa;
      const double* blk = s9 >= 4 ? sysn + (s9 - 4) * 21 : sys + static_cast<size_t>(qn) * kSysStride + (4 - s9) * 21;
      const double* pv = pub + 6 * static_cast<size_t>(qn);
#pragma unroll
      for (int c = 0; c < 6; c += 2) {
        b0 += __ldg(blk + ro[c]) * __ldg(pv + c);
        b1 += __ldg(blk + ro[c + 1]) * __ldg(pv + c + 1);
      }
    }
    b -= b0 + b1;
  }
  if (NLOC == 0) {
#pragma unroll
    for (int s9 = 0; s9 < 9; ++s9) {
      const int dx = s9 % 3 - 1, dy = s9 / 3 - 1;
      const int qa = na + dx, qb = nb + dy;
      const bool valid = act && qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh;
      const bool local = valid && qa >= alo && qa <= ahi && qb >= blo && qb <= bhi;
      const int qn = valid ? qb * a.gw + qa : 0;
      lidx[s9] = local ? 6 * ((ix + dx) + (iy + dy) * a.nxm) : 0;
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const double v = valid ? sys_entry(sys, G, n, qn, s9, r, c) : 0.0;
        arow[s9][c] = local ? v : 0.0;
        if (valid && !local && pub) b -= v * __ldg(pub + 6 * static_cast<size_t>(qn) + c);  // solver.cpp:437-448
      }
    }
  }
  // preconditioner of this unknown's field (solver.cpp:468-474)
  double m_self = 1.0, m_cross = 0.0;
  if (act) {
    const double* pre = sys + static_cast<size_t>(n) * kSysStride + kSysPre + 3 * (r >> 1);
    m_self = __ldg(pre + ((r & 1) ? 2 : 0));
    m_cross = __ldg(pre + 1);
  }
  auto apply = [&](double v) {  // local block SpMV (solver.cpp:452-467)
    if (TEAM == 32) __syncwarp(); else __syncthreads();
    psub[u] = v;
    if (TEAM == 32) __syncwarp(); else __syncthreads();
    double acc[3] = {0.0, 0.0, 0.0};  // three short chains instead of one long one
#pragma unroll
    for (int j = 0; j < NR; ++j)
#pragma unroll
      for (int c = 0; c < 6; ++c) acc[c % 3] += arow[j][c] * psub[lidx[j] + c];
    return act ? (acc[0] + acc[1]) + acc[2] : 0.0;
  };
  auto precond = [&](double rv) {
    const double partner = __shfl_xor_sync(0xffffffffu, rv, 1);
    return act ? m_self * rv + m_cross * partner : 0.0;
  };

  // pcg_impl (solver.cpp:320-361), warm start x0 = published
  double res = b - apply(x);
  double z = precond(res);
  double rz = team_sum<TEAM>(res * z, scratch);
  const double rz0 = fabs(rz);
  int flag = 0;
  if (rz0 != 0.0) {
    double p = z;
    for (int it = 0; it < a.pcg_iters; ++it) {
      const double ap = apply(p);
      const double pAp = team_sum<TEAM>(p * ap, scratch);
      if (pAp <= 0.0) {
        flag = kFlagCurvature;
        break;
      }
      const double alpha = rz / pAp;
      x += alpha * p;
      res -= alpha * ap;
      z = precond(res);
      const double rzn = team_sum<TEAM>(res * z, scratch);
      if (fabs(rzn) > 100.0 * rz0) {
        flag = kFlagGrowth;
        break;
      }
      const double beta = rzn / rz;
      rz = rzn;
      p = z + beta * p;
    }
  }
  if (!act) return;
  if (flag && u == 0) atomicOr(a.flags + pair, flag);
  const size_t o = (static_cast<size_t>(pair) * G + n) * 6 + r;
  if (a.last) {
    if (!isfinite(x)) atomicOr(a.flags + pair, kFlagStep);
    if ((a.active >> (r >> 1)) & 1) a.delta[o] += x;
    a.total[o] = a.base[o] + a.delta[o];
  } else {
    a.next[o] = x;
  }
}

// ---- k_schwarz22: 2x2-node subdomains (16 px tiles at grid step 8, the BASELINE cfg1-3 case) --------
// Same sweep as k_schwarz<32, 4>, but the subdomain's neighbourhood is staged in shared memory by
// bulk asynchronous copies (cp.async.bulk -> mbarrier) instead of ~90 scattered 8 B loads per lane:
// the system records of node rows b-1..b+1 x columns a-1..a+2 (every block the four rows touch
// lives there: forward slots in the own records, backward ones in the up/left neighbours') and
// the published x of rows b-1..b+2 x columns a-1..a+2. Lanes then read their rows from shared memory.
namespace bulk {
__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(b)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void copy(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(saddr(dst)), "l"(src), "r"(bytes), "r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(saddr(b)), "r"(phase) : "memory");
  } while (!done);
}
}  // namespace bulk

struct alignas(16) Swz22Smem {
  double rec[3][4][kSysStride];  // node rows b-1, b, b+1 x columns a-1 .. a+2
  double pub[4][4][6];           // published x, rows b-1 .. b+2 x columns a-1 .. a+2
  double psub[32];
  uint64_t bar;
};

// a / b for the PCG step lengths: the hardware reciprocal estimate refined by two Newton steps
// (error ~1 ulp against the correctly rounded quotient; no libdevice slow-path branch)
__device__ __forceinline__ double fdiv(double a, double b) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = __fma_rn(-b, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-b, r, 1.0);
  r = __fma_rn(r, e, r);
  return a * r;
}

struct Tile22 {  // one subdomain of the launch's range
  int pair, alo, ahi, blo, bhi;
};
__device__ __forceinline__ Tile22 tile22(const SwzArgs& a, int t, int nsub) {
  Tile22 T;
  T.pair = t / nsub;
  const int sub = a.sub0 + (t - T.pair * nsub);
  const int tx = sub % a.ntx, ty = sub / a.ntx;
  T.alo = (tx * a.tile + a.step - 1) / a.step;
  T.ahi = min(a.gw - 1, ((tx + 1) * a.tile - 1) / a.step);
  T.blo = (ty * a.tile + a.step - 1) / a.step;
  T.bhi = min(a.gh - 1, ((ty + 1) * a.tile - 1) / a.step);
  return T;
}

// Lane 0: arm the barrier with the tile's byte count and issue its bulk copies.
__device__ __forceinline__ void stage22(const SwzArgs& a, const Tile22& T, Swz22Smem& sm) {
  const size_t G = static_cast<size_t>(a.gw) * a.gh;
  const double* sys = a.sys + T.pair * G * kSysStride;
  const double* pubg = a.pub ? a.pub + T.pair * G * 6 : nullptr;
  const int c0 = max(T.alo - 1, 0);
  uint32_t bytes = 0;
  for (int ry = 0; ry < 3; ++ry) {
    const int row = T.blo - 1 + ry, c1 = min(T.alo + (ry == 2 ? 1 : 2), a.gw - 1);
    if (row >= 0 && row < a.gh && c1 >= c0) bytes += (c1 - c0 + 1) * kSysStride * 8;
  }
  if (pubg)
    for (int ry = 0; ry < 4; ++ry) {
      const int row = T.blo - 1 + ry, c1 = min(T.alo + 2, a.gw - 1);
      if (row >= 0 && row < a.gh && c1 >= c0) bytes += (c1 - c0 + 1) * 48;
    }
  bulk::mbar_expect(&sm.bar, bytes);
  for (int ry = 0; ry < 3; ++ry) {
    const int row = T.blo - 1 + ry, c1 = min(T.alo + (ry == 2 ? 1 : 2), a.gw - 1);
    if (row >= 0 && row < a.gh && c1 >= c0)
      bulk::copy(&sm.rec[ry][c0 - (T.alo - 1)][0], sys + (static_cast<size_t>(row) * a.gw + c0) * kSysStride,
                 (c1 - c0 + 1) * kSysStride * 8, &sm.bar);
  }
  if (pubg)
    for (int ry = 0; ry < 4; ++ry) {
      const int row = T.blo - 1 + ry, c1 = min(T.alo + 2, a.gw - 1);
      if (row >= 0 && row < a.gh && c1 >= c0)
        bulk::copy(&sm.pub[ry][c0 - (T.alo - 1)][0], pubg + (static_cast<size_t>(row) * a.gw + c0) * 6,
                   (c1 - c0 + 1) * 48, &sm.bar);
    }
}

// Persistent: each warp walks subdomains t = warp, warp + W, ...; the next subdomain's copies
// are issued as soon as the current one's rows are in registers, so they land during its PCG.
__global__ void __launch_bounds__(128) k_schwarz22(const SwzArgs a, int nsub, int total) {
  extern __shared__ __align__(16) unsigned char swz_raw[];
  const int team = threadIdx.x >> 5, u = threadIdx.x & 31;
  Swz22Smem& sm = reinterpret_cast<Swz22Smem*>(swz_raw)[team];
  const int W = gridDim.x * 4;
  int t = blockIdx.x * 4 + team;
  if (t >= total) return;
  const size_t G = static_cast<size_t>(a.gw) * a.gh;
  const int i = u / 6, r = u - 6 * (u / 6);
  const int ix = i & 1, iy = i >> 1;
  int ro[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) ro[c] = sym6(r, c);
  const bool has_pub = a.pub != nullptr;

  if (u == 0) bulk::mbar_init(&sm.bar);
  __syncwarp();
  Tile22 T = tile22(a, t, nsub);
  if (u == 0) stage22(a, T, sm);
  uint32_t phase = 0;
  for (; t < total; t += W) {
    const int na = T.alo + ix, nb = T.blo + iy;
    const bool act = u < 24 && na <= T.ahi && nb <= T.bhi;
    const int n = act ? nb * a.gw + na : 0;
    const int pair = T.pair;
    const int alo = T.alo, ahi = T.ahi, blo = T.blo, bhi = T.bhi;
    bulk::mbar_wait(&sm.bar, phase);
    phase ^= 1;

    const double* own = &sm.rec[1 + iy][1 + ix][0];
    double arow[4][6];
    double b = 0.0, x = 0.0;
    if (act) {
      b = own[kSysRhs + r];
      if (has_pub) x = sm.pub[1 + iy][1 + ix][r];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {  // dense local row over the tile's nodes
      const int jx = j & 1, jy = j >> 1;
      const bool ok = act && alo + jx <= ahi && blo + jy <= bhi;
      const int s9 = (jy - iy + 1) * 3 + (jx - ix + 1);
      const double* blk = s9 >= 4 ? own + (s9 - 4) * 21 : &sm.rec[1 + jy][1 + jx][0] + (4 - s9) * 21;
#pragma unroll
      for (int c = 0; c < 6; ++c) arow[j][c] = ok ? blk[ro[c]] : 0.0;
    }
    if (has_pub) {  // coupling to the frozen neighbours (solver.cpp:437-448), two alternating chains
      double b0 = 0.0, b1 = 0.0;
#pragma unroll
      for (int s9 = 0; s9 < 9; ++s9) {
        if (s9 == 4) continue;
        const int dx = s9 % 3 - 1, dy = s9 / 3 - 1;
        const int qa = na + dx, qb = nb + dy;
        const bool valid = act && qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh;
        const bool local = qa >= alo && qa <= ahi && qb >= blo && qb <= bhi;
        if (!valid || local) continue;
        const double* blk = s9 >= 4 ? own + (s9 - 4) * 21 : &sm.rec[1 + iy + dy][1 + ix + dx][0] + (4 - s9) * 21;
        const double* pv = &sm.pub[1 + iy + dy][1 + ix + dx][0];
#pragma unroll
        for (int c = 0; c < 6; c += 2) {
          b0 += blk[ro[c]] * pv[c];
          b1 += blk[ro[c + 1]] * pv[c + 1];
        }
      }
      b -= b0 + b1;
    }
    double m_self = 1.0, m_cross = 0.0;  // solver.cpp:468-474
    if (act) {
      const double* pre = own + kSysPre + 3 * (r >> 1);
      m_self = pre[(r & 1) ? 2 : 0];
      m_cross = pre[1];
    }
    // the staged rows are in registers: reuse the buffer for the next subdomain. Every lane orders its
    // generic reads of the buffer before the async-proxy writes of the next copies, then the warp syncs.
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (t + W < total) {
      T = tile22(a, t + W, nsub);
      if (u == 0) stage22(a, T, sm);
    }
    auto apply = [&](double v) {  // local block SpMV (solver.cpp:452-467)
      __syncwarp();
      sm.psub[u] = v;
      __syncwarp();
      double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[c % 3] += arow[j][c] * sm.psub[6 * j + c];
      return act ? (acc[0] + acc[1]) + acc[2] : 0.0;
    };
    auto precond = [&](double rv) {
      const double partner = __shfl_xor_sync(0xffffffffu, rv, 1);
      return act ? m_self * rv + m_cross * partner : 0.0;
    };
    // pcg_impl (solver.cpp:320-361), warm start x0 = published
    double res = b - apply(x);
    double z = precond(res);
    double rz = warp_sum(res * z);
    const double rz0 = fabs(rz);
    int flag = 0;
    if (rz0 != 0.0) {
      double p = z;
      for (int it = 0; it < a.pcg_iters; ++it) {
        const double ap = apply(p);
        const double pAp = warp_sum(p * ap);
        if (pAp <= 0.0) {
          flag = kFlagCurvature;
          break;
        }
        const double alpha = fdiv(rz, pAp);
        x += alpha * p;
        res -= alpha * ap;
        z = precond(res);
        const double rzn = warp_sum(res * z);
        if (fabs(rzn) > 100.0 * rz0) {
          flag = kFlagGrowth;
          break;
        }
        const double beta = fdiv(rzn, rz);
        rz = rzn;
        p = z + beta * p;
      }
    }
    if (flag && u == 0) atomicOr(a.flags + pair, flag);
    if (act) {
      const size_t o = (static_cast<size_t>(pair) * G + n) * 6 + r;
      if (a.last) {
        if (!isfinite(x)) atomicOr(a.flags + pair, kFlagStep);
        if ((a.active >> (r >> 1)) & 1) a.delta[o] += x;
        a.total[o] = a.base[o] + a.delta[o];
      } else {
        a.next[o] = x;
      }
    }
  }
}

constexpr int kPcgThreads = 1024;

__device__ double block_dot(const double* __restrict__ x, const double* __restrict__ y, int n, double* red) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i] * y[i];
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
  if (threadIdx.x < 32) t = warp_sum(t);
  __syncthreads();
  if (threadIdx.x == 0) red[32] = t;
  __syncthreads();
  return red[32];
}

__device__ void spmv(const double* __restrict__ sys, int gw, int gh, const double* __restrict__ x,
                     double* __restrict__ y) {
  const int G = gw * gh;
  for (int t = threadIdx.x; t < 6 * G; t += blockDim.x) {
    const int n = t / 6, r = t % 6, na = n % gw, nb = n / gw;
    double acc = 0.0;
    for (int s9 = 0; s9 < 9; ++s9) {
      const int qa = na + s9 % 3 - 1, qb = nb + s9 / 3 - 1;
      if (qa < 0 || qa >= gw || qb < 0 || qb >= gh) continue;
      const int qn = qb * gw + qa;
      for (int c = 0; c < 6; ++c) acc += sys_entry(sys, G, n, qn, s9, r, c) * x[6 * qn + c];
    }
    y[t] = acc;
  }
}

__device__ void precondition(const double* __restrict__ sys, int G, const double* __restrict__ r,
                             double* __restrict__ z) {
  for (int t = threadIdx.x; t < 6 * G; t += blockDim.x) {
    const int n = t / 6, k = t % 6;
    const double* pre = sys + static_cast<size_t>(n) * kSysStride + kSysPre + 3 * (k >> 1);
    const int e = t & ~1;
    z[t] = (k & 1) ? pre[1] * r[e] + pre[2] * r[e + 1] : pre[0] * r[e] + pre[1] * r[e + 1];
  }
}

__global__ void __launch_bounds__(kPcgThreads) k_pcg_global(const PcgArgs a) {
  __shared__ double red[33];
  const int pair = blockIdx.x;
  const int G = a.gw * a.gh, M = 6 * G;
  const double* sys = a.sys + static_cast<size_t>(pair) * G * kSysStride;
  double* x = a.x + static_cast<size_t>(pair) * M;
  double* r = a.r + static_cast<size_t>(pair) * M;
  double* z = a.z + static_cast<size_t>(pair) * M;
  double* p = a.p + static_cast<size_t>(pair) * M;
  double* ap = a.ap + static_cast<size_t>(pair) * M;
  double* tr = a.trace ? a.trace + static_cast<size_t>(pair) * (a.iters + 1) : nullptr;
  for (int t = threadIdx.x; t < M; t += blockDim.x) {
    x[t] = 0.0;
    r[t] = __ldg(sys + static_cast<size_t>(t / 6) * kSysStride + kSysRhs + t % 6);
  }
  __syncthreads();
  if (tr) {
    const double nr = block_dot(r, r, M, red);
    if (threadIdx.x == 0) tr[0] = sqrt(nr);
  }
  precondition(sys, G, r, z);
  __syncthreads();
  double rz = block_dot(r, z, M, red);
  const double rz0 = fabs(rz);
  int flag = 0;
  if (rz0 == 0.0) {
    if (tr && threadIdx.x == 0)
      for (int it = 0; it < a.iters; ++it) tr[it + 1] = 0.0;
  } else {
    for (int t = threadIdx.x; t < M; t += blockDim.x) p[t] = z[t];
    __syncthreads();
    for (int it = 0; it < a.iters; ++it) {
      spmv(sys, a.gw, a.gh, p, ap);
      __syncthreads();
      const double pAp = block_dot(p, ap, M, red);
      if (pAp <= 0.0) {
        flag = kFlagCurvature;
        break;
      }
      const double alpha = rz / pAp;
      for (int t = threadIdx.x; t < M; t += blockDim.x) {
        x[t] += alpha * p[t];
        r[t] -= alpha * ap[t];
      }
      __syncthreads();
      if (tr) {
        const double nr = block_dot(r, r, M, red);
        if (threadIdx.x == 0) tr[it + 1] = sqrt(nr);
      }
      precondition(sys, G, r, z);
      __syncthreads();
      const double rzn = block_dot(r, z, M, red);
      if (fabs(rzn) > 100.0 * rz0) {
        flag = kFlagGrowth;
        break;
      }
      const double beta = rzn / rz;
      rz = rzn;
      for (int t = threadIdx.x; t < M; t += blockDim.x) p[t] = z[t] + beta * p[t];
      __syncthreads();
    }
  }
  if (flag && threadIdx.x == 0) atomicOr(a.flags + pair, flag);
  __syncthreads();
  if (a.update) {
    const size_t o = static_cast<size_t>(pair) * M;
    bool bad = false;
    for (int t = threadIdx.x; t < M; t += blockDim.x) {
      bad = bad || !isfinite(x[t]);
      if ((a.active >> ((t % 6) >> 1)) & 1) a.delta[o + t] += x[t];
      a.total[o + t] = a.base[o + t] + a.delta[o + t];
    }
    if (bad) atomicOr(a.flags + pair, kFlagStep);
  }
}

// ---- k_pcg_cluster: the same global PCG with a thread-block cluster per pair -------------------------
// k_pcg_global runs one CTA per pair, so a batch smaller than the SM count leaves most of the GPU idle.
// Here a cluster of kPcgCluster CTAs shares one pair. Each CTA owns a contiguous node slice of every
// vector. Dots reduce per CTA in a fixed order, then every CTA sums the kPcgCluster partials in rank
// order through distributed shared memory, so all CTAs hold the same bits. Cluster barriers
// (release/acquire) make each CTA's slice of p visible to the others' SpMV.
constexpr int kPcgCluster = 8, kPcgClusterThreads = 256;

__device__ double slice_dot(const double* __restrict__ x, const double* __restrict__ y, int lo, int hi, double* red,
                            double* part, cg::cluster_group& cl) {
  double s = 0.0;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) s += x[i] * y[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
    *part = t;
  }
  cl.sync();
  double tot = 0.0;
  for (int k = 0; k < kPcgCluster; ++k) tot += *cl.map_shared_rank(part, k);
  return tot;
}

__global__ void __cluster_dims__(kPcgCluster, 1, 1) __launch_bounds__(kPcgClusterThreads)
    k_pcg_cluster(const PcgArgs a) {
  __shared__ double red[kPcgClusterThreads / 32];
  __shared__ double part[2];  // alternating dot partials (a partial is rewritten two dots later)
  cg::cluster_group cl = cg::this_cluster();
  const int rank = static_cast<int>(cl.block_rank());
  const int pair = blockIdx.x / kPcgCluster;
  const int G = a.gw * a.gh, M = 6 * G;
  const int lo = 6 * static_cast<int>(static_cast<long long>(G) * rank / kPcgCluster);
  const int hi = 6 * static_cast<int>(static_cast<long long>(G) * (rank + 1) / kPcgCluster);
  const double* sys = a.sys + static_cast<size_t>(pair) * G * kSysStride;
  double* x = a.x + static_cast<size_t>(pair) * M;
  double* r = a.r + static_cast<size_t>(pair) * M;
  double* z = a.z + static_cast<size_t>(pair) * M;
  double* p = a.p + static_cast<size_t>(pair) * M;
  double* ap = a.ap + static_cast<size_t>(pair) * M;
  double* tr = a.trace ? a.trace + static_cast<size_t>(pair) * (a.iters + 1) : nullptr;
  int nd = 0;  // dots issued (selects the partial slot)
  auto dot = [&](const double* u, const double* v) { return slice_dot(u, v, lo, hi, red, &part[nd++ & 1], cl); };
  auto spmv_slice = [&](const double* xv, double* y) {  // rows [lo, hi) of the 9-slot block SpMV
    for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) {
      const int n = t / 6, rr = t % 6, na = n % a.gw, nb = n / a.gw;
      double acc = 0.0;
      for (int s9 = 0; s9 < 9; ++s9) {
        const int qa = na + s9 % 3 - 1, qb = nb + s9 / 3 - 1;
        if (qa < 0 || qa >= a.gw || qb < 0 || qb >= a.gh) continue;
        const int qn = qb * a.gw + qa;
        for (int c = 0; c < 6; ++c) acc += sys_entry(sys, G, n, qn, s9, rr, c) * xv[6 * qn + c];
      }
      y[t] = acc;
    }
  };
  auto precond_slice = [&]() {
    for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) {
      const int n = t / 6, k = t % 6;
      const double* pre = sys + static_cast<size_t>(n) * kSysStride + kSysPre + 3 * (k >> 1);
      const int e = t & ~1;
      z[t] = (k & 1) ? pre[1] * r[e] + pre[2] * r[e + 1] : pre[0] * r[e] + pre[1] * r[e + 1];
    }
  };
  for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) {
    x[t] = 0.0;
    r[t] = __ldg(sys + static_cast<size_t>(t / 6) * kSysStride + kSysRhs + t % 6);
  }
  __syncthreads();
  if (tr) {
    const double nr = dot(r, r);
    if (rank == 0 && threadIdx.x == 0) tr[0] = sqrt(nr);
  }
  precond_slice();
  __syncthreads();
  double rz = dot(r, z);
  const double rz0 = fabs(rz);
  int flag = 0;
  if (rz0 == 0.0) {
    if (tr && rank == 0 && threadIdx.x == 0)
      for (int it = 0; it < a.iters; ++it) tr[it + 1] = 0.0;
  } else {
    for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) p[t] = z[t];
    cl.sync();  // every slice of p is written before any SpMV reads it
    for (int it = 0; it < a.iters; ++it) {
      spmv_slice(p, ap);
      __syncthreads();
      const double pAp = dot(p, ap);
      if (pAp <= 0.0) {
        flag = kFlagCurvature;
        break;
      }
      const double alpha = rz / pAp;
      for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) {
        x[t] += alpha * p[t];
        r[t] -= alpha * ap[t];
      }
      __syncthreads();
      if (tr) {
        const double nr = dot(r, r);
        if (rank == 0 && threadIdx.x == 0) tr[it + 1] = sqrt(nr);
      }
      precond_slice();
      __syncthreads();
      const double rzn = dot(r, z);
      if (fabs(rzn) > 100.0 * rz0) {
        flag = kFlagGrowth;
        break;
      }
      const double beta = rzn / rz;
      rz = rzn;
      // (every slice's SpMV of this iteration read p before the pAp dot's cluster barrier)
      for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) p[t] = z[t] + beta * p[t];
      cl.sync();  // the new p is complete
    }
  }
  if (flag && rank == 0 && threadIdx.x == 0) atomicOr(a.flags + pair, flag);
  if (a.update) {
    const size_t o = static_cast<size_t>(pair) * M;
    bool bad = false;
    for (int t = lo + threadIdx.x; t < hi; t += blockDim.x) {
      bad = bad || !isfinite(x[t]);
      if ((a.active >> ((t % 6) >> 1)) & 1) a.delta[o + t] += x[t];
      a.total[o + t] = a.base[o + t] + a.delta[o + t];
    }
    if (bad) atomicOr(a.flags + pair, kFlagStep);
  }
  cl.sync();  // no CTA leaves while a partner may still read its shared partials
}

}  // namespace

void init_solve_attributes() {
  cudaFuncSetAttribute(k_schwarz22, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * sizeof(Swz22Smem));
}

void launch_schwarz(const SwzArgs& a_in, int B, cudaStream_t s) {
  SwzArgs a = a_in;
  if (a.sub1 <= 0) {  // whole level
    a.sub0 = 0;
    a.sub1 = a.ntx * a.nty;
  }
  const int nsub = a.sub1 - a.sub0;
  if (nsub <= 0) return;
  const int nodes = a.nxm * a.nym;
  static const bool use22 = [] {
    const char* e = std::getenv("HWF_SWZ22");
    return !e || std::atoi(e) != 0;
  }();
  if (use22 && a.nxm == 2 && a.nym == 2) {
    static const int grid_cap = [] {
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_schwarz22, 128, 4 * sizeof(Swz22Smem));
      return std::max(1, sms * std::max(per_sm, 1));
    }();
    const int total = nsub * B;
    const int grid = std::min(grid_cap, (total + 3) / 4);
    k_schwarz22<<<grid, 128, 4 * sizeof(Swz22Smem), s>>>(a, nsub, total);
  } else if (nodes <= 4) {
    k_schwarz<32, 4><<<dim3((nsub + 3) / 4, B), 128, 0, s>>>(a);
  } else if (6 * nodes <= 128) {
    k_schwarz<128, 0><<<dim3(nsub, B), 128, 0, s>>>(a);
  } else if (6 * nodes <= 384) {
    k_schwarz<384, 0><<<dim3(nsub, B), 384, 0, s>>>(a);
  } else {
    k_schwarz<1024, 0><<<dim3(nsub, B), 1024, 0, s>>>(a);
  }
}

void launch_pcg_global(const PcgArgs& a, int B, cudaStream_t s) {
  static const int sms = [] {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
  }();
  if (B < sms)  // fewer pairs than SMs: a cluster of CTAs per pair
    k_pcg_cluster<<<B * kPcgCluster, kPcgClusterThreads, 0, s>>>(a);
  else
    k_pcg_global<<<B, kPcgThreads, 0, s>>>(a);
}

}  // namespace hwf
