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
// k_pcg_init / k_pcg_spmv / k_pcg_update: the subdomain_px = 0 mode (pcg_solve,
// solver.cpp:365-380), tiled over the whole GPU with fixed-order dots (see below).
#include <algorithm>
#include <cstdlib>


#include "launch.h"

namespace hwf {
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
#ifdef HWF_EXACT_MATH
  return a / b;
#endif
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

// ---- global PCG (subdomain_px = 0; pcg_solve, solver.cpp:365-380; pcg_impl, :320-361) ---------------
// One kernel per phase, each spread over (tiles, pairs):
//   k_pcg_init    x = 0, r = b, z = M r, p = 0                              partials r.z, r.r
//   k_pcg_spmv    p = z + beta p (tile and halo, staged in shared memory), Ap   partial p.Ap
//   k_pcg_update  x += alpha p, r -= alpha Ap, z = M r                     partials r.z, r.r
// A tile is a segment of 32 nodes of one grid row: one warp, one node per lane. The system is
// entry-major ([entry][node], written so by k_node in this mode), so a lane's 21 loads of a block
// are 256 B coalesced rows across the warp. Every dot is the same fixed tree: per node
// ((u0v0 + u1v1) + (u2v2 + u3v3)) + (u4v4 + u5v5) rounded op by op, an xor tree over the 32 lanes,
// then the pair's tiles in index order (strided over 128 threads, xor trees, the 4 warps in order),
// summed by whichever CTA of the pair finishes last, which leaves the scalars (rz, alpha, beta,
// stop) in `state`. The order depends only on the level's tiling: results are bitwise independent
// of the batch size. A pair that meets a divergence condition stops iterating (flag set) and still
// applies its step at the end. (A fused all-iterations variant, one CTA or an 8-CTA cluster per
// pair, was slower at every level size measured.)
constexpr int kPcgTile = 32, kPcgWarps = 4, kPcgThreads = 32 * kPcgWarps;
enum : int { kStRz = 0, kStRz0, kStAlpha, kStBeta, kStStop, kStCount = 8 };
constexpr int kPhCols = kPcgTile + 4;

struct PcgTile {
  int b, a0, width;
  bool live;
};
__device__ __forceinline__ int pcg_ntiles(int gw, int gh) { return (gw + kPcgTile - 1) / kPcgTile * gh; }
__device__ __forceinline__ PcgTile pcg_tile_at(int gw, int gh, int tile, int t_end) {
  const int tpr = (gw + kPcgTile - 1) / kPcgTile, nt = tpr * gh;
  PcgTile T;
  T.live = tile < min(nt, t_end);
  const int t = T.live ? tile : nt - 1;
  T.b = t / tpr;
  T.a0 = (t - T.b * tpr) * kPcgTile;
  T.width = T.live ? min(kPcgTile, gw - T.a0) : 0;
  return T;
}

__device__ __forceinline__ double node_dot(const double (&u)[6], const double (&v)[6]) {
  const double s01 = __dadd_rn(__dmul_rn(u[0], v[0]), __dmul_rn(u[1], v[1]));
  const double s23 = __dadd_rn(__dmul_rn(u[2], v[2]), __dmul_rn(u[3], v[3]));
  const double s45 = __dadd_rn(__dmul_rn(u[4], v[4]), __dmul_rn(u[5], v[5]));
  return __dadd_rn(__dadd_rn(s01, s23), s45);
}

// Sum of the pair's tile partials part[k * stride], k < n, in the canonical order; every thread
// of the CTA returns the same value.
__device__ __forceinline__ double pair_total(const double* part, int n, int stride, double* red) {
  double s = 0.0;
  for (int k = threadIdx.x; k < n; k += kPcgThreads) s += __ldcg(part + static_cast<size_t>(k) * stride);
  s = warp_sum(s);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kPcgWarps; ++w) t += red[w];
  return t;
}

// Publishes this CTA's partials and reports whether it is the pair's last CTA to do so.
__device__ __forceinline__ bool pcg_last_cta(unsigned* count, int nctas, int* sflag) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) *sflag = atomicAdd(count, 1u) == static_cast<unsigned>(nctas - 1);
  __syncthreads();
  const bool last = *sflag != 0;
  if (last) {
    __threadfence();
    if (threadIdx.x == 0) *count = 0;  // ready for the next kernel
  }
  return last;
}

struct PcgPtr {
  const double* sys;  // entry-major: entry e of node n at sys[e * G + n]
  double *x, *r, *z, *ap, *p, *p2, *part, *st;
  unsigned* cnt;
  double* tr;
  size_t G;
  int ntiles;
};
__device__ __forceinline__ PcgPtr pcg_ptr(const PcgArgs& a, int pair) {
  const size_t G = static_cast<size_t>(a.gw) * a.gh, M = 6 * G;
  PcgPtr P;
  P.G = G;
  P.ntiles = pcg_ntiles(a.gw, a.gh);
  P.sys = a.sys + pair * G * kSysStride;
  P.x = a.x + pair * M;
  P.r = a.r + pair * M;
  P.z = a.z + pair * M;
  P.ap = a.ap + pair * M;
  P.p = a.p + pair * M;
  P.p2 = a.p2 + pair * M;
  P.part = a.part + static_cast<size_t>(pair) * P.ntiles * 2;
  P.st = a.state + static_cast<size_t>(pair) * kStCount;
  P.cnt = a.count + pair;
  P.tr = a.trace ? a.trace + static_cast<size_t>(pair) * (a.iters + 1) : nullptr;
  return P;
}

__device__ __forceinline__ void ld6(const double* p, double (&v)[6]) {
  const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double2 t = __ldcg(q + i);
    v[2 * i] = t.x;
    v[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ void st6(double* p, const double (&v)[6]) {
  double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
  for (int i = 0; i < 3; ++i) q[i] = make_double2(v[2 * i], v[2 * i + 1]);
}

// z = M r (solver.cpp:468-474 via NormalSystem::precond_block): the node's three 2x2 blocks
// (split in two so callers can issue the nine loads before their stores: the compiler cannot move
// them across stores it cannot prove disjoint)
__device__ __forceinline__ void pcg_precond_load(const PcgPtr& P, size_t n, double (&M)[9]) {
#pragma unroll
  for (int i = 0; i < 9; ++i) M[i] = __ldg(P.sys + (kSysPre + i) * P.G + n);
}
__device__ __forceinline__ void pcg_precond_apply(const double (&M)[9], const double (&r)[6], double (&z)[6]) {
#pragma unroll
  for (int f = 0; f < 3; ++f) {
    const double m0 = M[3 * f], m1 = M[3 * f + 1], m2 = M[3 * f + 2];
    z[2 * f] = m0 * r[2 * f] + m1 * r[2 * f + 1];
    z[2 * f + 1] = m1 * r[2 * f] + m2 * r[2 * f + 1];
  }
}
__device__ __forceinline__ void pcg_precond(const PcgPtr& P, size_t n, const double (&r)[6], double (&z)[6]) {
  double M[9];
  pcg_precond_load(P, n, M);
  pcg_precond_apply(M, r, z);
}

// Tile partial of one per-node value (xor tree over the warp); every lane returns it.
__device__ __forceinline__ double tile_partial(bool act, double v) { return warp_sum(act ? v : 0.0); }

__device__ __forceinline__ size_t tile_node(const PcgArgs& a, const PcgTile& T, int j) {
  return static_cast<size_t>(T.b) * a.gw + T.a0 + min(j, max(T.width - 1, 0));
}

// ---- per-tile phases (one warp each) ----
__device__ __forceinline__ void tile_init(const PcgArgs& a, const PcgPtr& P, const PcgTile& T, double& prz,
                                          double& prr) {
  const int j = threadIdx.x & 31;
  const bool act = j < T.width;
  const size_t n = tile_node(a, T, j);
  double r[6], z[6];
#pragma unroll
  for (int k = 0; k < 6; ++k) r[k] = act ? __ldg(P.sys + (kSysRhs + k) * P.G + n) : 0.0;
  pcg_precond(P, n, r, z);
  if (act) {
    const double zero[6] = {0, 0, 0, 0, 0, 0};
    st6(P.x + 6 * n, zero);
    st6(P.r + 6 * n, r);
    st6(P.z + 6 * n, z);
    st6(P.p + 6 * n, zero);
    // strip split: the search direction of the halo rows starts at zero here too (tile_spmv keeps it)
    if (T.b == a.row_lo && a.row_lo > 0) st6(P.p + 6 * (n - a.gw), zero);
    if (T.b == a.row_hi - 1 && a.row_hi < a.gh) st6(P.p + 6 * (n + a.gw), zero);
  }
  prz = tile_partial(act, node_dot(r, z));
  prr = tile_partial(act, node_dot(r, r));
}

// p_next = z + beta p_prev over the tile and its one-node halo (this warp's shared memory,
// field-major so lane j reads consecutive words), then Ap = A p_next with the 9-slot block SpMV.
__device__ __forceinline__ double tile_spmv(const PcgArgs& a, const PcgPtr& P, const PcgTile& T, double beta,
                                            const double* __restrict__ p_prev, double* __restrict__ p_next,
                                            double (*ph)[6][kPhCols]) {
  const int j = threadIdx.x & 31;
  const bool act = j < T.width;
  const int a_ = T.a0 + min(j, max(T.width - 1, 0));
  const size_t n = static_cast<size_t>(T.b) * a.gw + a_;
  // block s9 of this node's row: forward slots from its own record, backward ones as the
  // neighbour's forward block; invalid slots read the own record (never used) so every load is
  // unconditional and the next block's loads can be in flight during this block's FMAs
  auto block = [&](int s9, bool& valid) -> const double* {
    const int dx = s9 % 3 - 1, dy = s9 / 3 - 1;
    const int qa = a_ + dx, qb = T.b + dy;
    valid = act && qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh;
    const size_t nq = s9 >= 4 || !valid ? n : static_cast<size_t>(qb) * a.gw + qa;
    return P.sys + static_cast<size_t>(s9 >= 4 ? s9 - 4 : 4 - s9) * 21 * P.G + nq;
  };
  double A[2][21];
  bool vb[9];
#ifdef HWF_DIAG_SPMV_FWD_ONLY  // diagnostic A/B only (wrong results): the 5 forward slots, no backward blocks
  constexpr int s9_first = 4;
#else
  constexpr int s9_first = 0;
#endif
  {
    const double* b0 = block(s9_first, vb[s9_first]);
#pragma unroll
    for (int m = 0; m < 21; ++m) A[s9_first & 1][m] = __ldg(b0 + m * P.G);
  }
  // stage p_next = z + beta p_prev, rows b-1..b+1 x nodes a0-1 .. a0+width (6 (width + 2) contiguous
  // doubles per row), all of a row's loads issued before its stores
  const int span = 6 * (T.width + 2);
  __syncwarp();
#pragma unroll
  for (int row = 0; row < 3; ++row) {
    const int qb = T.b - 1 + row;
    constexpr int kPer = (6 * (kPcgTile + 2) + 31) / 32;
    double zz[kPer], pp[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = j + 32 * k, col = i / 6, c = i - 6 * col, qa = T.a0 - 1 + col;
      const bool ok = i < span && qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh;
      const size_t o = ok ? 6 * (static_cast<size_t>(qb) * a.gw + qa) + c : 0;
      zz[k] = ok ? __ldcg(P.z + o) : 0.0;
      pp[k] = ok ? __ldcg(p_prev + o) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int i = j + 32 * k, col = i / 6, c = i - 6 * col, qa = T.a0 - 1 + col;
      if (i >= span) continue;
      const bool ok = qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh;
      const double v = ok ? zz[k] + beta * pp[k] : 0.0;  // p = z + beta p (solver.cpp:358)
      ph[row][c][col] = v;
    }
  }
  __syncwarp();
  // p_next to global only now, from shared memory: global stores inside the staging would keep the
  // compiler from hoisting the later rows' loads. The own row; in a strip split also the halo rows,
  // which the neighbouring rank owns (the same z + beta p from the exchanged z, so only z crosses ranks).
  if (act) {
#pragma unroll
    for (int row = 0; row < 3; ++row) {
      const bool keep = row == 1 || (row == 0 && T.b == a.row_lo && a.row_lo > 0) ||
                        (row == 2 && T.b == a.row_hi - 1 && a.row_hi < a.gh);
      if (!keep) continue;
      double pr[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) pr[c] = ph[row][c][j + 1];
      st6(p_next + 6 * (n + static_cast<long long>(row - 1) * a.gw), pr);
    }
  }
  double acc[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int s9 = s9_first; s9 < 9; ++s9) {  // NormalSystem::apply (solver.cpp:80-98)
    if (s9 + 1 < 9) {
      const double* bn = block(s9 + 1, vb[s9 + 1]);
#pragma unroll
      for (int m = 0; m < 21; ++m) A[(s9 + 1) & 1][m] = __ldg(bn + m * P.G);
    }
    if (!vb[s9]) continue;
    const int dx = s9 % 3 - 1, dy = s9 / 3 - 1;
    double pv[6];
#pragma unroll
    for (int c = 0; c < 6; ++c) pv[c] = ph[1 + dy][c][j + 1 + dx];
#pragma unroll
    for (int i = 0; i < 6; ++i)
#pragma unroll
      for (int c = 0; c < 6; ++c) acc[i] += A[s9 & 1][sym6(i, c)] * pv[c];
  }
  double pown[6];
#pragma unroll
  for (int c = 0; c < 6; ++c) pown[c] = ph[1][c][j + 1];
  if (act) st6(P.ap + 6 * n, acc);
  return tile_partial(act, node_dot(pown, acc));
}

__device__ __forceinline__ void tile_update(const PcgArgs& a, const PcgPtr& P, const PcgTile& T, double alpha,
                                            const double* __restrict__ p_cur, bool want_rr, double& prz, double& prr) {
  const int j = threadIdx.x & 31;
  const bool act = j < T.width;
  const size_t n = tile_node(a, T, j);
  double r[6] = {0, 0, 0, 0, 0, 0}, z[6], M[9];
  pcg_precond_load(P, n, M);
  if (act) {
    double x[6], p[6], ap[6];
    ld6(P.x + 6 * n, x);
    ld6(p_cur + 6 * n, p);
    ld6(P.r + 6 * n, r);
    ld6(P.ap + 6 * n, ap);
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      x[k] += alpha * p[k];  // solver.cpp:348-349
      r[k] -= alpha * ap[k];
    }
    st6(P.x + 6 * n, x);
    st6(P.r + 6 * n, r);
  }
  pcg_precond_apply(M, r, z);
  if (act) st6(P.z + 6 * n, z);
  prz = tile_partial(act, node_dot(r, z));
  prr = want_rr ? tile_partial(act, node_dot(r, r)) : 0.0;
}

// delta += x, total = base + delta (solver.cpp:518-523); returns whether any x is non-finite.
__device__ __forceinline__ bool tile_apply(const PcgArgs& a, const PcgPtr& P, const PcgTile& T, int pair) {
  const int j = threadIdx.x & 31;
  bool bad = false;
  if (j < T.width) {
    const size_t n = tile_node(a, T, j);
    const size_t o = static_cast<size_t>(pair) * 6 * P.G + 6 * n;
#pragma unroll
    for (int k = 0; k < 6; ++k) {
      const double xv = __ldcg(P.x + 6 * n + k);
      bad = bad || !isfinite(xv);
      if ((a.active >> (k >> 1)) & 1) a.delta[o + k] += xv;
      a.total[o + k] = a.base[o + k] + a.delta[o + k];
    }
  }
  return __any_sync(0xffffffffu, bad);
}

// Pair totals -> scalars (the last CTA of a phase, or k_pcg_scalars after a split's all-gather).
__device__ __forceinline__ void finish_init(const PcgArgs& a, const PcgPtr& P, double* red) {
  const double rz = pair_total(P.part, P.ntiles, 2, red);
  const double rr = pair_total(P.part + 1, P.ntiles, 2, red);
  if (threadIdx.x == 0) {
    if (P.tr) P.tr[0] = sqrt(rr);
    P.st[kStRz] = rz;
    P.st[kStRz0] = fabs(rz);
    P.st[kStBeta] = 0.0;
    P.st[kStStop] = rz == 0.0 ? 1.0 : 0.0;  // early return (solver.cpp:334-338)
    if (rz == 0.0 && P.tr)
      for (int it = 0; it < a.iters; ++it) P.tr[it + 1] = 0.0;
  }
}
__device__ __forceinline__ void finish_spmv(const PcgArgs& a, const PcgPtr& P, int pair, double* red) {
  const double pAp = pair_total(P.part, P.ntiles, 2, red);
  if (threadIdx.x == 0) {
    if (pAp <= 0.0) {  // solver.cpp:344-346
      P.st[kStStop] = 1.0;
      atomicOr(a.flags + pair, kFlagCurvature);
    } else {
      P.st[kStAlpha] = P.st[kStRz] / pAp;
    }
  }
}
__device__ __forceinline__ void finish_update(const PcgArgs& a, const PcgPtr& P, int pair, int it, double* red) {
  const double rzn = pair_total(P.part, P.ntiles, 2, red);
  const double rr = P.tr ? pair_total(P.part + 1, P.ntiles, 2, red) : 0.0;
  if (threadIdx.x == 0) {
    if (P.tr) P.tr[it + 1] = sqrt(rr);
    if (fabs(rzn) > 100.0 * P.st[kStRz0]) {  // solver.cpp:352-355
      P.st[kStStop] = 1.0;
      atomicOr(a.flags + pair, kFlagGrowth);
    } else {
      P.st[kStBeta] = rzn / P.st[kStRz];
      P.st[kStRz] = rzn;
    }
  }
}

__global__ void __launch_bounds__(kPcgThreads) k_pcg_init(const PcgArgs a) {
  __shared__ double red[kPcgWarps];
  __shared__ int sflag;
  const int pair = blockIdx.y, tile = a.t0 + blockIdx.x * kPcgWarps + (threadIdx.x >> 5);
  const PcgPtr P = pcg_ptr(a, pair);
  const PcgTile T = pcg_tile_at(a.gw, a.gh, tile, a.t1);
  double prz, prr;
  tile_init(a, P, T, prz, prr);
  if ((threadIdx.x & 31) == 0 && T.live) {
    P.part[2 * tile] = prz;
    P.part[2 * tile + 1] = prr;
  }
  if (!a.split && pcg_last_cta(P.cnt, gridDim.x, &sflag)) finish_init(a, P, red);
  if (a.iters == 0 && a.update) {
    __syncthreads();
    if (tile_apply(a, P, T, pair) && (threadIdx.x & 31) == 0) atomicOr(a.flags + pair, kFlagStep);
  }
}

__global__ void __launch_bounds__(kPcgThreads, 4) k_pcg_spmv(const PcgArgs a, int it) {
  __shared__ double ph_all[kPcgWarps][3][6][kPhCols];
  __shared__ double red[kPcgWarps];
  __shared__ int sflag;
  const int pair = blockIdx.y, tile = a.t0 + blockIdx.x * kPcgWarps + (threadIdx.x >> 5);
  const PcgPtr P = pcg_ptr(a, pair);
  if (__ldcg(P.st + kStStop) != 0.0) return;
  const PcgTile T = pcg_tile_at(a.gw, a.gh, tile, a.t1);
  const double* prev = it & 1 ? P.p2 : P.p;
  double* next = it & 1 ? P.p : P.p2;
  const double part = tile_spmv(a, P, T, __ldcg(P.st + kStBeta), prev, next, ph_all[threadIdx.x >> 5]);
  if ((threadIdx.x & 31) == 0 && T.live) P.part[2 * tile] = part;
  if (!a.split && pcg_last_cta(P.cnt, gridDim.x, &sflag)) finish_spmv(a, P, pair, red);
}

__global__ void __launch_bounds__(kPcgThreads) k_pcg_update(const PcgArgs a, int it) {
  __shared__ double red[kPcgWarps];
  __shared__ int sflag;
  const int pair = blockIdx.y, tile = a.t0 + blockIdx.x * kPcgWarps + (threadIdx.x >> 5);
  const PcgPtr P = pcg_ptr(a, pair);
  const PcgTile T = pcg_tile_at(a.gw, a.gh, tile, a.t1);
  const bool final_step = a.update && it == a.iters - 1;
  if (__ldcg(P.st + kStStop) == 0.0) {
    double prz, prr;
    tile_update(a, P, T, __ldcg(P.st + kStAlpha), it & 1 ? P.p : P.p2, P.tr != nullptr, prz, prr);
    if ((threadIdx.x & 31) == 0 && T.live) {
      P.part[2 * tile] = prz;
      P.part[2 * tile + 1] = prr;
    }
    if (!a.split && pcg_last_cta(P.cnt, gridDim.x, &sflag)) finish_update(a, P, pair, it, red);
  }
  if (final_step && tile_apply(a, P, T, pair) && (threadIdx.x & 31) == 0) atomicOr(a.flags + pair, kFlagStep);
}

// Strip split: the scalars of a phase from the all-gathered partials of every rank (same tree).
__global__ void __launch_bounds__(kPcgThreads) k_pcg_scalars(const PcgArgs a, int phase, int it) {
  __shared__ double red[kPcgWarps];
  const int pair = blockIdx.x;
  const PcgPtr P = pcg_ptr(a, pair);
  if (phase == 0) {
    finish_init(a, P, red);
  } else if (__ldcg(P.st + kStStop) == 0.0) {
    if (phase == 1) finish_spmv(a, P, pair, red);
    else finish_update(a, P, pair, it, red);
  }
}

// Small levels (every tile of a pair fits one CTA: <= 16 tiles): the whole pcg_solve of a pair in ONE CTA, a
// warp per tile exactly as the per-phase kernels map them, so every per-node value, every tile partial (warp xor
// tree) and every pair total (pair_total's order over the partials, here in shared memory) is the same double as
// theirs; the phases meet at __syncthreads instead of kernel boundaries and last-CTA atomics (11 launches per GN
// iteration at these levels were latency, not work). x, r, z, Ap and the preconditioner stay in registers; p lives
// in shared memory, where the 9-slot SpMV reads the neighbours' values; the system is read from global (L2).
constexpr int kFusedMaxTiles = 16;  // 512 threads: 128 registers, no spills
__device__ __forceinline__ double pair_total_smem(const double* part, int n, int stride, double* red) {
  // pair_total's summation order (128-thread stride, xor trees, the 4 warps in order) over shared memory
  double s = 0.0;
  if (threadIdx.x < kPcgThreads)
    for (int k = threadIdx.x; k < n; k += kPcgThreads) s += part[k * stride];
  s = warp_sum(s);
  __syncthreads();
  if (threadIdx.x < kPcgThreads && (threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kPcgWarps; ++w) t += red[w];
  __syncthreads();  // red and part reusable
  return t;
}

// SYS_SMEM (the smallest levels, whose pair's system fits): the system is staged in shared memory once and the
// five iterations read it there.
template <bool SYS_SMEM>
__global__ void __launch_bounds__(32 * kFusedMaxTiles) k_pcg_fused(const PcgArgs a) {
  extern __shared__ __align__(16) double fsm[];
  const int pair = blockIdx.x, tile = threadIdx.x >> 5, j = threadIdx.x & 31;
  const PcgPtr P = pcg_ptr(a, pair);
  double* ps = fsm;                         // p, node-major [G][6]
  double* part = fsm + 6 * P.G;             // [ntiles][2]
  double* red = part + 2 * kFusedMaxTiles;  // [kPcgWarps]
  double* sys_s = red + kPcgWarps;          // SYS_SMEM: the pair's system, entry-major [kSysStride][G]
  __shared__ uint64_t sys_bar;
  if (SYS_SMEM) {  // one bulk-async (TMA) copy of the pair's contiguous 960 G bytes, completing on an mbarrier
    if (threadIdx.x == 0) bulk::mbar_init(&sys_bar);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t bytes = static_cast<uint32_t>(kSysStride * sizeof(double) * P.G);
      bulk::mbar_expect(&sys_bar, bytes);
      bulk::copy(sys_s, P.sys, bytes, &sys_bar);
    }
    bulk::mbar_wait(&sys_bar, 0);
  }
  const double* S = SYS_SMEM ? sys_s : P.sys;
  auto lds = [&](const double* q) { return SYS_SMEM ? *q : __ldg(q); };

  const PcgTile T = pcg_tile_at(a.gw, a.gh, tile, P.ntiles);
  const bool act = j < T.width;
  const int a_ = T.a0 + min(j, max(T.width - 1, 0));
  const size_t n = static_cast<size_t>(T.b) * a.gw + a_;
  const bool want_rr = P.tr != nullptr;
  auto precond = [&](const double (&rv)[6], double (&zv)[6]) {  // pcg_precond from S
    double M[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) M[i] = lds(S + (kSysPre + i) * P.G + n);
    pcg_precond_apply(M, rv, zv);
  };
  // k_pcg_init
  double r[6], z[6], x[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int k = 0; k < 6; ++k) r[k] = act ? lds(S + (kSysRhs + k) * P.G + n) : 0.0;
  precond(r, z);  // (the preconditioner is re-read per update: fewer live registers)
  for (int i = threadIdx.x; i < 6 * static_cast<int>(P.G); i += blockDim.x) ps[i] = 0.0;  // p_prev = 0
  {
    const double prz = tile_partial(act, node_dot(r, z)), prr = tile_partial(act, node_dot(r, r));
    if (j == 0 && T.live) {
      part[2 * tile] = prz;
      part[2 * tile + 1] = prr;
    }
  }
  __syncthreads();
  double rz = pair_total_smem(part, P.ntiles, 2, red);
  const double rr0 = pair_total_smem(part + 1, P.ntiles, 2, red);
  const double rz0 = fabs(rz);
  double beta = 0.0, alpha = 0.0;
  bool stop = rz == 0.0;  // solver.cpp:334-338
  if (threadIdx.x == 0 && P.tr) {
    P.tr[0] = sqrt(rr0);
    if (stop)
      for (int it = 0; it < a.iters; ++it) P.tr[it + 1] = 0.0;
  }
  for (int it = 0; it < a.iters && !stop; ++it) {
    // k_pcg_spmv: p = z + beta p (solver.cpp:358), then Ap over the 9 slots in the per-phase kernel's order
    double pown[6];
    if (act) {
#pragma unroll
      for (int c = 0; c < 6; ++c) pown[c] = z[c] + beta * ps[6 * n + c];
    }
    __syncthreads();  // every neighbour has read the previous p
    if (act) {
#pragma unroll
      for (int c = 0; c < 6; ++c) ps[6 * n + c] = pown[c];
    }
    __syncthreads();
    double acc[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll 1
    for (int s9 = 0; s9 < 9; ++s9) {  // NormalSystem::apply (solver.cpp:80-98)
      const int dx = s9 % 3 - 1, dy = s9 / 3 - 1;
      const int qa = a_ + dx, qb = T.b + dy;
      if (!(act && qa >= 0 && qa < a.gw && qb >= 0 && qb < a.gh)) continue;
      const size_t nq = static_cast<size_t>(qb) * a.gw + qa;
      const double* blk = S + static_cast<size_t>(s9 >= 4 ? s9 - 4 : 4 - s9) * 21 * P.G + (s9 >= 4 ? n : nq);
      double A[21];
#pragma unroll
      for (int m = 0; m < 21; ++m) A[m] = lds(blk + m * P.G);
      double pv[6];
#pragma unroll
      for (int c = 0; c < 6; ++c) pv[c] = ps[6 * nq + c];
#pragma unroll
      for (int i = 0; i < 6; ++i)
#pragma unroll
        for (int c = 0; c < 6; ++c) acc[i] += A[sym6(i, c)] * pv[c];
    }
    if (!act) {
#pragma unroll
      for (int c = 0; c < 6; ++c) pown[c] = 0.0;
    }
    {
      const double pp = tile_partial(act, node_dot(pown, acc));
      if (j == 0 && T.live) part[2 * tile] = pp;
    }
    __syncthreads();
    const double pAp = pair_total_smem(part, P.ntiles, 2, red);
    if (pAp <= 0.0) {  // solver.cpp:344-346
      if (threadIdx.x == 0) atomicOr(a.flags + pair, kFlagCurvature);
      stop = true;
      break;
    }
    alpha = rz / pAp;
    // k_pcg_update: x += alpha p, r -= alpha Ap, z = M r (solver.cpp:348-351)
    if (act) {
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        x[k] += alpha * pown[k];
        r[k] -= alpha * acc[k];
      }
    }
    precond(r, z);
    {
      const double prz = tile_partial(act, node_dot(r, z));
      const double prr = want_rr ? tile_partial(act, node_dot(r, r)) : 0.0;
      if (j == 0 && T.live) {
        part[2 * tile] = prz;
        part[2 * tile + 1] = prr;
      }
    }
    __syncthreads();
    const double rzn = pair_total_smem(part, P.ntiles, 2, red);
    const double rr = want_rr ? pair_total_smem(part + 1, P.ntiles, 2, red) : 0.0;
    if (threadIdx.x == 0 && P.tr) P.tr[it + 1] = sqrt(rr);
    if (fabs(rzn) > 100.0 * rz0) {  // solver.cpp:352-355
      if (threadIdx.x == 0) atomicOr(a.flags + pair, kFlagGrowth);
      stop = true;
      break;
    }
    beta = rzn / rz;
    rz = rzn;
  }
  if (act) st6(P.x + 6 * n, x);  // the hwf_pcg seam reads x back
  if (a.update) {  // delta += x, total = base + delta (solver.cpp:518-523), as tile_apply
    bool bad = false;
    if (act) {
      const size_t o = static_cast<size_t>(pair) * 6 * P.G + 6 * n;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        bad = bad || !isfinite(x[k]);
        if ((a.active >> (k >> 1)) & 1) a.delta[o + k] += x[k];
        a.total[o + k] = a.base[o + k] + a.delta[o + k];
      }
    }
    if (__any_sync(0xffffffffu, bad) && j == 0) atomicOr(a.flags + pair, kFlagStep);
  }
}

}  // namespace

void init_solve_attributes() {
  cudaFuncSetAttribute(k_schwarz22, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * sizeof(Swz22Smem));
  cudaFuncSetAttribute(k_pcg_fused<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_pcg_fused<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
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

int pcg_tiles(int gw, int gh) { return (gw + kPcgTile - 1) / kPcgTile * gh; }

namespace {
PcgArgs whole(const PcgArgs& in) {
  PcgArgs a = in;
  if (a.t1 <= 0) {
    a.t0 = 0;
    a.t1 = pcg_tiles(a.gw, a.gh);
    a.row_lo = 0;
    a.row_hi = a.gh;
  }
  return a;
}
dim3 pcg_grid(const PcgArgs& a, int B) {
  return dim3(static_cast<unsigned>(std::max(1, (a.t1 - a.t0 + kPcgWarps - 1) / kPcgWarps)), static_cast<unsigned>(B));
}
}  // namespace

#ifndef HWF_PCG_FUSED  // small levels run pcg_solve in one CTA per pair (A/B knob: 0 = per-phase kernels everywhere)
#define HWF_PCG_FUSED 1
#endif
#ifndef HWF_PCG_SYS_SMEM  // ... with the pair's system staged in shared memory when it fits (A/B knob)
#define HWF_PCG_SYS_SMEM 1
#endif
size_t pcg_fused_smem(int gw, int gh, bool sys_smem = false) {
  return (static_cast<size_t>(6 + (sys_smem ? kSysStride : 0)) * gw * gh + 2 * kFusedMaxTiles + kPcgWarps) *
         sizeof(double);
}
void launch_pcg_global(const PcgArgs& a_in, int B, cudaStream_t s) {
  const PcgArgs a = whole(a_in);
  const int ntiles = pcg_tiles(a.gw, a.gh);
  if (HWF_PCG_FUSED && !a.split && ntiles <= kFusedMaxTiles && pcg_fused_smem(a.gw, a.gh) <= 200 * 1024) {
    // at least kPcgWarps warps: pair_total's tree reads the partial of each of the first 4 (tile-less warps add 0)
    if (HWF_PCG_SYS_SMEM && pcg_fused_smem(a.gw, a.gh, true) <= 200 * 1024)
      k_pcg_fused<true><<<B, 32 * std::max(ntiles, kPcgWarps), pcg_fused_smem(a.gw, a.gh, true), s>>>(a);
    else
      k_pcg_fused<false><<<B, 32 * std::max(ntiles, kPcgWarps), pcg_fused_smem(a.gw, a.gh), s>>>(a);
    return;
  }
  const dim3 grid = pcg_grid(a, B);
  k_pcg_init<<<grid, kPcgThreads, 0, s>>>(a);
  for (int it = 0; it < a.iters; ++it) {
    k_pcg_spmv<<<grid, kPcgThreads, 0, s>>>(a, it);
    k_pcg_update<<<grid, kPcgThreads, 0, s>>>(a, it);
  }
}
void launch_pcg_phase(const PcgArgs& a_in, int phase, int it, cudaStream_t s) {
  const PcgArgs a = whole(a_in);
  if (a.t1 <= a.t0) return;  // this rank owns no rows at this level
  const dim3 grid = pcg_grid(a, 1);
  if (phase == 0) k_pcg_init<<<grid, kPcgThreads, 0, s>>>(a);
  else if (phase == 1) k_pcg_spmv<<<grid, kPcgThreads, 0, s>>>(a, it);
  else k_pcg_update<<<grid, kPcgThreads, 0, s>>>(a, it);
}
void launch_pcg_scalars(const PcgArgs& a_in, int phase, int it, cudaStream_t s) {
  k_pcg_scalars<<<1, kPcgThreads, 0, s>>>(whole(a_in), phase, it);
}
int pcg_launches(int gw, int gh, int iters) {
  if (HWF_PCG_FUSED && pcg_tiles(gw, gh) <= kFusedMaxTiles && pcg_fused_smem(gw, gh) <= 200 * 1024) return 1;
  return 1 + 2 * iters;
}

}  // namespace hwf
