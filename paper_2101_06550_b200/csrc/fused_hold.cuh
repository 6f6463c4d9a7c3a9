// fused_hold.cuh — the shared-LHS batched solve with every tile HELD ON CHIP
// between its two sweeps: the production path of pent_solve / tri_solve /
// pent_solve_many / pent_solve_strided, the ADI sweeps and the 1D CH step
// whenever the systems fit a cluster (n <= CSM * NW * Q rows).
//
// Same tiles, sweeps and carry algebra as fused_cluster.cuh (a 64-row chunk
// of 32 systems, lane = system; P1 = zero-inflow forward sweep + carries,
// P2 = sweeps from the true inflows), but consumer warp w of
// cluster CTA c OWNS chunk q = c*cpc + w for every group the cluster solves:
//   * its tile goes from the TMA slot into registers once, P1 runs on it, the
//     warp waits for the group's carry scan (cluster_scan: one DSMEM exchange),
//     and P2 runs on the SAME registers -- f is read from HBM exactly once and
//     x written once (the two-pass design re-reads f through L2; on B200 that
//     re-read, not HBM, bounded it);
//   * the slot is refilled with the warp's chunk of the cluster's NEXT group
//     as soon as the tile is in registers, so one group of loads is always in
//     flight behind the sweeps and the scan (NW tiles per SM);
//   * the chunk's coefficient rows are the same for every group: loaded into
//     the warp's private shared memory once per launch.
// The carry records and the DSMEM exchange are those of fused_cluster.cuh (the
// scan runs on warp 0 after its own P1: every warp waits for it anyway); a CTA's warps are never more than one group apart (P2 of
// group t needs every warp's P1 of t), so two record parities suffice.
#pragma once
#include "fused_cluster.cuh"

namespace pb {
namespace fh {

using namespace fs;
using fc::CArgs;

constexpr int NW = 8;                // warps = chunks per CTA per group (warp 0 also runs the scan)
constexpr int NTHREADS = 32 * NW;    // 2 warps per SM sub-partition: the full 255-register budget each
template <int MODE>
constexpr int csmax() { return MODE == MODE_CH1D ? 8 : 16; }   // cluster size (16: non-portable)

template <typename T, int MODE>
struct HCfg {
    static constexpr int TILE = Q * TW;
    static constexpr int HALO = MODE == MODE_CH1D ? TW * 2 : 0;
    static constexpr int E1K = 1024 / (int)sizeof(T);
    static constexpr int SLOT = (TILE + HALO + E1K - 1) / E1K * E1K;   // 1 KB multiple (swizzle)
};

template <typename T, int MODE>
struct HSmem {
    using C = HCfg<T, MODE>;
    static constexpr int CSM = csmax<MODE>();
    // one record parity: warp w alone writes (P1) and reads (P2) rec[0][w], and
    // the scan rewrites it only once every warp's P1 of the next group is in
    static constexpr int NPAR = 1;
    T slot[NW][C::SLOT];
    T park[Q][TW];                   // warp 0's tile while it runs the scan
    T coef[NW][Q * COEF_STRIDE];     // the warp's chunk: F0 F1 F2 - B1 B2 Z1 Z2 per row
    T wab[NW][Q * 2];                // and its back-substitution functional rows (W_a, W_b)
    T rec[NPAR][NW][TW][4];          // (yF0, yF1, zB0, zB1) -> (yin0, yin1, zin0, zin1)
    T spec[NPAR][4][TW];
    T xl[NPAR][TW][2];
    T xa[CSM][TW][2], xb[CSM][TW][2];
    T yv[CSM][TW][2];
    T xP[CSM][12];
    T xg[4][TW], xr[4][2];
    T phi[NW][8];
    T ct[NW][12];                    // this CTA's chunk maps
    T rsp[8];
    uint64_t full[NW];
    uint64_t p1done[2], scandone[2];
    uint64_t xch, xcons;
};

// P1 on the tile column in registers: zero-inflow forward sweep, carry (y0, y1)
// and back-substitution functional (a0, a1).  SPEC: the tile holds cyclic
// rows -- always among the last four rows of the system, hence among the last
// four valid rows of the tile -- whose zero-inflow g go to gs (a four-entry
// ring indexed by the unrolled row, read once after the sweep).  FULL: kmax == Q.
template <typename T, int K, bool SPEC, bool FULL>
__device__ __forceinline__ void p1_sweep(const T (&v)[Q], const T *cp, const T *wp, int kmax, int64_t r0,
                                         const int64_t (&srow)[4], T &y0, T &y1, T &a0, T &a1, T (&gs)[4])
{
    y0 = y1 = a0 = a1 = T(0);
    T hist[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        if (FULL || k < kmax) {
            T f0, f1, f2, fz, wa, wb;
            lds2(cp + k * COEF_STRIDE, f0, f1);
            lds2(cp + k * COEF_STRIDE + 2, f2, fz);
            lds2(wp + 2 * k, wa, wb);
            T tt = f0 * v[k];
            if (K == 2) tt -= f2 * y0;
            const T gg = tt - f1 * y1;   // newest carry last: one FMA on the chain
            y0 = y1;
            y1 = gg;
            a0 += wa * gg;
            a1 += wb * gg;
            if (SPEC) hist[k & 3] = gg;
        }
    }
    if (SPEC) {
#pragma unroll
        for (int jx = 0; jx < 4; ++jx) {
            const int64_t rr = srow[jx] - r0;
            if (srow[jx] >= 0 && rr >= 0 && rr < kmax) {
                const int j = (int)(rr & 3);
                gs[jx] = j == 0 ? hist[0] : j == 1 ? hist[1] : j == 2 ? hist[2] : hist[3];
            }
        }
    }
}

// Full-tile sweeps with the coefficient rows software-pipelined PD rows ahead
// (the shared-memory latency, ~30 cycles, is otherwise exposed on every row:
// the tile column leaves the compiler no registers to hoist loads on its own).
constexpr int PD = 4;

template <typename T, int K, bool SPEC>
__device__ __forceinline__ void p1_full(const T (&v)[Q], const T *cp, const T *wp, T &y0, T &y1, T &a0, T &a1,
                                        T (&hist)[4])
{
    T c01[PD][2], c2[PD][2], cw[PD][2];
#pragma unroll
    for (int k = 0; k < PD; ++k) {
        lds2(cp + k * COEF_STRIDE, c01[k][0], c01[k][1]);
        lds2(cp + k * COEF_STRIDE + 2, c2[k][0], c2[k][1]);
        lds2(wp + 2 * k, cw[k][0], cw[k][1]);
    }
    y0 = y1 = a0 = a1 = T(0);
#pragma unroll
    for (int k = 0; k < Q; ++k) {
        const int sl = k % PD;
        const T f0 = c01[sl][0], f1 = c01[sl][1], f2 = c2[sl][0], wa = cw[sl][0], wb = cw[sl][1];
        if (k + PD < Q) {
            lds2(cp + (k + PD) * COEF_STRIDE, c01[sl][0], c01[sl][1]);
            lds2(cp + (k + PD) * COEF_STRIDE + 2, c2[sl][0], c2[sl][1]);
            lds2(wp + 2 * (k + PD), cw[sl][0], cw[sl][1]);
        }
        T tt = f0 * v[k];
        if (K == 2) tt -= f2 * y0;
        const T gg = tt - f1 * y1;   // newest carry last: one FMA on the chain
        y0 = y1;
        y1 = gg;
        a0 += wa * gg;
        a1 += wb * gg;
        if (SPEC) hist[k & 3] = gg;
    }
}

// P2 on a full tile: forward sweep from (y0, y1); back substitution from
// (z0, z1) with the cyclic correction x - Z x_l folded into the same pass.
template <typename T, int K, bool PER>
__device__ __forceinline__ void p2_full(T (&v)[Q], const T *cp, T y0, T y1, T z0, T z1, T xl0, T xl1)
{
    {
        T c01[PD][2], c2[PD][2];
#pragma unroll
        for (int k = 0; k < PD; ++k) {
            lds2(cp + k * COEF_STRIDE, c01[k][0], c01[k][1]);
            lds2(cp + k * COEF_STRIDE + 2, c2[k][0], c2[k][1]);
        }
#pragma unroll
        for (int k = 0; k < Q; ++k) {
            const int sl = k % PD;
            const T f0 = c01[sl][0], f1 = c01[sl][1], f2 = c2[sl][0];
            if (k + PD < Q) {
                lds2(cp + (k + PD) * COEF_STRIDE, c01[sl][0], c01[sl][1]);
                lds2(cp + (k + PD) * COEF_STRIDE + 2, c2[sl][0], c2[sl][1]);
            }
            T t = f0 * v[k];
            if (K == 2) t -= f2 * y0;
            const T g = t - f1 * y1;
            y0 = y1;
            y1 = g;
            v[k] = g;
        }
    }
    T cb[PD][2], cz[PD][2];
#pragma unroll
    for (int j = 0; j < PD; ++j) {
        const int k = Q - 1 - j;
        lds2(cp + k * COEF_STRIDE + 4, cb[j][0], cb[j][1]);
        if (PER) lds2(cp + k * COEF_STRIDE + 6, cz[j][0], cz[j][1]);
    }
#pragma unroll
    for (int j = 0; j < Q; ++j) {
        const int k = Q - 1 - j, sl = j % PD;
        const T b1 = cb[sl][0], b2 = cb[sl][1], z1v = PER ? cz[sl][0] : T(0), z2v = PER ? cz[sl][1] : T(0);
        if (j + PD < Q) {
            lds2(cp + (k - PD) * COEF_STRIDE + 4, cb[sl][0], cb[sl][1]);
            if (PER) lds2(cp + (k - PD) * COEF_STRIDE + 6, cz[sl][0], cz[sl][1]);
        }
        T t = v[k];
        if (K == 2) t -= b2 * z1;
        const T xx = t - b1 * z0;
        z1 = z0;
        z0 = xx;
        if (PER) {
            T o = xx - z1v * xl0;   // cyclic correction (Navon eq:solve / Sherman–Morrison)
            if (K == 2) o -= z2v * xl1;
            v[k] = o;
        } else {
            v[k] = xx;
        }
    }
}

// ---------------------------------------------------------------- the carry scan of one group (warp 0)
// The fold of fused_cluster.cuh's cluster_scan with everything in registers
// (at most NW chunks per CTA, unrolled; the tile is parked in shared memory
// meanwhile) and a PULL exchange: every CTA writes its summary into its own
// shared memory, signals the cluster once, and loads the peers' summaries
// with independent DSMEM loads (one round trip, not one per peer).
//   chunk i:   yin0_i = y (zero CTA inflow), c0_i = zB_i + H_i y,  y <- Mf_i y + yF_i
//   CTA:       a = y_out, P = prod Mf, b = backward fold of c0 with Mb,
//              Pb = prod Mb, Kc = sum_i (Mb_0..Mb_{i-1}) H_i Phi_i (b's response to Y)
//   cluster:   Y_{v+1} = P_v Y_v + a_v;  Z_v = Z above v, Z <- Pb_v Z + Kc_v Y_v + b_v
__device__ __forceinline__ void ldc2(uint32_t a, double &x, double &y)
{
    asm volatile("ld.shared::cluster.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void ldc2(uint32_t a, float &x, float &y)
{
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a) : "memory");
}
__device__ __forceinline__ void ldc1(uint32_t a, double &x)
{
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(x) : "r"(a) : "memory");
}
__device__ __forceinline__ void ldc1(uint32_t a, float &x)
{
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(x) : "r"(a) : "memory");
}

template <typename T, int K, bool PER, int CSM, typename SM>
__device__ __forceinline__ void hold_scan(const CArgs<T> &A, SM &S, int t, int c, int q0, int nch, int lane)
{
    const bool multi = A.cs > 1;
    int li[4];   // local chunk of each cyclic row (-1: not mine)
#pragma unroll
    for (int jx = 0; jx < 4; ++jx) {
        const int64_t qq = A.srow[jx] >= 0 ? A.srow[jx] / Q - q0 : -1;
        li[jx] = PER && qq >= 0 && qq < nch ? (int)qq : -1;
    }
    T y0 = T(0), y1 = T(0);
    T P[4] = {T(1), T(0), T(0), T(1)}, Qb[4] = {T(1), T(0), T(0), T(1)}, Kc[4] = {T(0), T(0), T(0), T(0)};
    T yi[NW][2], cz[NW][2];
    T gj[4] = {T(0), T(0), T(0), T(0)}, rj[4][2] = {{T(0), T(0)}, {T(0), T(0)}, {T(0), T(0)}, {T(0), T(0)}};
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        yi[i][0] = yi[i][1] = cz[i][0] = cz[i][1] = T(0);
        if (i < nch) {
            const T mf[4] = {S.ct[i][0], S.ct[i][1], S.ct[i][2], S.ct[i][3]};
            const T h[4] = {S.ct[i][8], S.ct[i][9], S.ct[i][10], S.ct[i][11]};
            T t0, t1;
            yi[i][0] = y0, yi[i][1] = y1;
            mv(h, y0, y1, t0, t1);
            cz[i][0] = S.rec[0][i][lane][2] + t0;
            cz[i][1] = S.rec[0][i][lane][3] + t1;
            if (PER) {
#pragma unroll
                for (int jx = 0; jx < 4; ++jx)
                    if (li[jx] == i) {
                        gj[jx] = S.spec[0][jx][lane] + S.rsp[jx * 2] * y0 + S.rsp[jx * 2 + 1] * y1;
                        rj[jx][0] = S.rsp[jx * 2] * P[0] + S.rsp[jx * 2 + 1] * P[2];
                        rj[jx][1] = S.rsp[jx * 2] * P[1] + S.rsp[jx * 2 + 1] * P[3];
                    }
            }
            mv(mf, y0, y1, t0, t1);
            y0 = t0 + S.rec[0][i][lane][0];
            y1 = t1 + S.rec[0][i][lane][1];
            if (multi) {
                // Kc += Qb H_i Phi_i ; Qb <- Qb Mb_i ; Phi <- Mf_i Phi  (lane-uniform)
                const T mb[4] = {S.ct[i][4], S.ct[i][5], S.ct[i][6], S.ct[i][7]};
                T hp[4], qh[4];
                mmul(h, P, hp);
                mmul(Qb, hp, qh);
#pragma unroll
                for (int e = 0; e < 4; ++e) Kc[e] += qh[e];
                mmul(Qb, mb, Qb);
                mmul(mf, P, P);
            }
        }
    }
    T b0 = T(0), b1 = T(0);
#pragma unroll
    for (int i = NW - 1; i >= 0; --i) {
        if (i < nch) {
            const T mb[4] = {S.ct[i][4], S.ct[i][5], S.ct[i][6], S.ct[i][7]};
            T t0, t1;
            mv(mb, b0, b1, t0, t1);
            b0 = t0 + cz[i][0];
            b1 = t1 + cz[i][1];
        }
    }
    T Zc0 = T(0), Zc1 = T(0), y1c = b0, y2c = b1;   // one CTA: Y = Z = 0, (x_0, x_1) = my outflow
    T gv[4] = {gj[0], gj[1], gj[2], gj[3]};
    if (multi) {
        const int cs = A.cs;
        // ---- publish (once every peer has read my previous summary)
        if (t >= 1) fc::wait_cluster(&S.xcons, (uint32_t)((t - 1) & 1));
        S.xa[c][lane][0] = y0, S.xa[c][lane][1] = y1;
        S.xb[c][lane][0] = b0, S.xb[c][lane][1] = b1;
        if (lane < 4) S.xP[c][lane] = P[lane], S.xP[c][4 + lane] = Qb[lane], S.xP[c][8 + lane] = Kc[lane];
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx)
                if (li[jx] >= 0) {
                    S.xg[jx][lane] = gj[jx];
                    if (lane < 2) S.xr[jx][lane] = rj[jx][lane];
                }
        }
        fc::fence_cluster();
        __syncwarp();
        if (lane < cs) fc::arrive_remote(&S.xch, lane);
        fc::wait_cluster(&S.xch, (uint32_t)(t & 1));
        // ---- pull: every peer's summary into my copies (all loads issued before
        // the first use: one DSMEM round trip)
#pragma unroll
        for (int r0 = 0; r0 < CSM; r0 += 8) {
            if (r0 < cs) {
                T la[8][4], lp[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int r = r0 + u;
                    if (r < cs && r != c) {
                        ldc2(fc::mapa(&S.xa[r][lane][0], r), la[u][0], la[u][1]);
                        ldc2(fc::mapa(&S.xb[r][lane][0], r), la[u][2], la[u][3]);
                        if (lane < 12) ldc1(fc::mapa(&S.xP[r][lane], r), lp[u]);
                    }
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int r = r0 + u;
                    if (r < cs && r != c) {
                        S.xa[r][lane][0] = la[u][0], S.xa[r][lane][1] = la[u][1];
                        S.xb[r][lane][0] = la[u][2], S.xb[r][lane][1] = la[u][3];
                        if (lane < 12) S.xP[r][lane] = lp[u];
                    }
                }
            }
        }
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx) {
                const int ow = A.srow[jx] >= 0 ? (int)(A.srow[jx] / Q) / A.cpc : c;
                if (ow != c) {
                    T g;
                    ldc1(fc::mapa(&S.xg[jx][lane], ow), g);
                    S.xg[jx][lane] = g;
                    if (lane < 2) {
                        ldc1(fc::mapa(&S.xr[jx][lane], ow), g);
                        S.xr[jx][lane] = g;
                    }
                }
            }
        }
        __syncwarp();
        if (lane < cs) fc::arrive_remote(&S.xcons, lane);   // this group's summaries consumed
        // ---- every CTA's forward inflow Y_v, then backward inflows from the top
        {
            T ya = T(0), yb = T(0);
            for (int v = 0; v < cs; ++v) {
                S.yv[v][lane][0] = ya, S.yv[v][lane][1] = yb;
                T t0, t1;
                mv(S.xP[v], ya, yb, t0, t1);
                ya = t0 + S.xa[v][lane][0];
                yb = t1 + S.xa[v][lane][1];
            }
        }
        T Za = T(0), Zb = T(0);
        for (int v = cs - 1; v >= 0; --v) {
            if (v == c) Zc0 = Za, Zc1 = Zb;
            T t0, t1, u0, u1;
            mv(S.xP[v] + 4, Za, Zb, t0, t1);
            mv(S.xP[v] + 8, S.yv[v][lane][0], S.yv[v][lane][1], u0, u1);
            Za = t0 + u0 + S.xb[v][lane][0];
            Zb = t1 + u1 + S.xb[v][lane][1];
        }
        y1c = Za, y2c = Zb;
        if (PER) {
#pragma unroll
            for (int jx = 0; jx < 4; ++jx)
                if (A.srow[jx] >= 0) {
                    const int ow = (int)(A.srow[jx] / Q) / A.cpc;
                    gv[jx] = S.xg[jx][lane] + S.xr[jx][0] * S.yv[ow][lane][0] + S.xr[jx][1] * S.yv[ow][lane][1];
                }
        }
        // ---- my chunks: yin_i += Phi_i Y, c_i += H_i Phi_i Y
        const T Y0 = S.yv[c][lane][0], Y1 = S.yv[c][lane][1];
        T Ph[4] = {T(1), T(0), T(0), T(1)};
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            if (i < nch) {
                const T mf[4] = {S.ct[i][0], S.ct[i][1], S.ct[i][2], S.ct[i][3]};
                const T h[4] = {S.ct[i][8], S.ct[i][9], S.ct[i][10], S.ct[i][11]};
                T t0, t1, hp[4];
                mv(Ph, Y0, Y1, t0, t1);
                yi[i][0] += t0;
                yi[i][1] += t1;
                mmul(h, Ph, hp);
                mv(hp, Y0, Y1, t0, t1);
                cz[i][0] += t0;
                cz[i][1] += t1;
                mmul(mf, Ph, Ph);
            }
        }
    }
    // ---- zin walk from Z_c; records -> (yin, zin)
    T z0 = Zc0, z1 = Zc1;
#pragma unroll
    for (int i = NW - 1; i >= 0; --i) {
        if (i < nch) {
            const T mb[4] = {S.ct[i][4], S.ct[i][5], S.ct[i][6], S.ct[i][7]};
            S.rec[0][i][lane][0] = yi[i][0];
            S.rec[0][i][lane][1] = yi[i][1];
            S.rec[0][i][lane][2] = z0;
            S.rec[0][i][lane][3] = z1;
            T t0, t1;
            mv(mb, z0, z1, t0, t1);
            z0 = t0 + cz[i][0];
            z1 = t1 + cz[i][1];
        }
    }
    if (!PER) return;
    // ---- cyclic pair: (x_0, x_1) = the system's first two unknowns; x_l
    const double *sc = A.scal;
    T xl0, xl1;
    if (K == 2) {
        // Navon (eq:first_two)
        const T ym1 = gv[1], ym2 = gv[0] - T(sc[10]) * gv[1];
        const T qa = gv[2] - (T(sc[4]) * y1c + T(sc[5]) * ym2 + T(sc[6]) * ym1);
        const T qb = gv[3] - (T(sc[7]) * y1c + T(sc[8]) * y2c + T(sc[9]) * ym1);
        xl0 = T(sc[0]) * qa + T(sc[1]) * qb;
        xl1 = T(sc[2]) * qa + T(sc[3]) * qb;
    } else {
        // Sherman–Morrison
        xl0 = (y1c + T(sc[0]) * gv[0]) / T(sc[1]);
        xl1 = T(0);
    }
    S.xl[0][lane][0] = xl0;
    S.xl[0][lane][1] = xl1;
}

template <typename T, int K, bool PER, int MODE, int LAY>
__global__ void __launch_bounds__(NTHREADS, 1) fh_kernel(const __grid_constant__ CUtensorMap tmap, const CArgs<T> A)
{
    using C = HCfg<T, MODE>;
    constexpr int TILE = C::TILE;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1 KB aligned (the 128B swizzle of contiguous tiles); derived from smem_raw
    // by pointer arithmetic so the compiler keeps the shared address space
    HSmem<T, MODE> &sm = *reinterpret_cast<HSmem<T, MODE> *>(smem_raw + ((1024u - (su32(smem_raw) & 1023u)) & 1023u));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c = (int)cg::this_cluster().block_rank();
    const int cl = blockIdx.x / A.cs;                         // cluster index
    const int q0 = c * A.cpc, nch = max(0, min(A.cpc, A.nq - q0));   // this CTA's chunks
    const int T_ = cl < A.G ? (A.G - 1 - cl) / A.ncl + 1 : 0;   // groups of this cluster
    if (threadIdx.x == 0) {
        for (int i = 0; i < NW; ++i) bar_init(&sm.full[i], 1);
        for (int p = 0; p < 2; ++p) {
            bar_init(&sm.p1done[p], nch);
            bar_init(&sm.scandone[p], 1);
        }
        bar_init(&sm.xch, A.cs);
        bar_init(&sm.xcons, A.cs);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cg::this_cluster().sync();   // barriers initialised cluster-wide before any remote arrive

    // every CTA owns >= 1 chunk (the launcher's CS is minimal), so warp 0 exists
    if (warp < nch) {
        {
            const int q = q0 + warp;
            const int64_t r0 = (int64_t)q * Q;
            const int kmax = (int)min((int64_t)Q, A.n - r0);
            T *slot = sm.slot[warp];
            uint64_t *full = &sm.full[warp];
            const uint64_t pol = policy_evict_first();
            // the next group's tile (and, MODE_CH1D, its two halo rows) into the slot
            auto issue = [&](int t) {
                const int g = cl + t * A.ncl;
                const int b = g / A.Gb, gl = g - b * A.Gb;
                bar_expect_tx(full, (uint32_t)((TILE + C::HALO) * sizeof(T)));
                if (LAY == LAY_CONTIG) {
#pragma unroll
                    for (int bx = 0; bx < Q / Sw<T>::EB; ++bx) {
                        T *dst = slot + bx * TW * Sw<T>::EB;
                        const int r = (int)r0 + bx * Sw<T>::EB;
                        if (A.flat) tma_load2(dst, &tmap, r, (int)((int64_t)b * A.M + gl * TW), full, pol);
                        else tma_load3(dst, &tmap, r, gl * TW, b, full, pol);
                    }
                } else if (A.flat) {
                    tma_load2(slot, &tmap, gl * TW, (int)((int64_t)b * A.n + r0), full, pol);
                } else {
                    tma_load3(slot, &tmap, gl * TW, (int)r0, b, full, pol);
                }
                if (MODE == MODE_CH1D) {
                    const T *ub = A.x + (int64_t)b * A.bstride + (int64_t)gl * TW;
                    const int64_t rlo = r0 == 0 ? A.n - 1 : r0 - 1, rhi = r0 + kmax == A.n ? 0 : r0 + kmax;
                    bulk_load(slot + TILE, ub + rlo * A.pitch, TW * sizeof(T), full);
                    bulk_load(slot + TILE + TW, ub + rhi * A.pitch, TW * sizeof(T), full);
                }
            };
            if (lane == 0 && T_ > 0) issue(0);
            // the chunk's coefficient rows, once
            T *cp = sm.coef[warp], *wp = sm.wab[warp];
            for (int e = lane; e < kmax * COEF_STRIDE; e += 32) cp[e] = A.coef[r0 * COEF_STRIDE + e];
            for (int k = lane; k < kmax; k += 32) {
                wp[2 * k] = A.rec[(r0 + k) * REC + 3];
                wp[2 * k + 1] = A.rec[(r0 + k) * REC + 4];
            }
            if (warp == 0) {
                // the CTA's chunk maps and cyclic responses for the scan
                for (int e = lane; e < nch * 12; e += 32) sm.ct[e / 12][e % 12] = A.ct[(int64_t)q0 * 12 + e];
                if (lane < 8) sm.rsp[lane] = A.rsp[lane];
            }
            __syncwarp();
            const bool spec_tile = PER && q >= A.srow[0] / Q;
#ifdef FH_PROF
            long long pacc[16] = {0};
            long long _t = clock64();
            long long *pt = pacc + 8;
#define FHQ(i) do { long long _n = clock64(); pacc[i] += _n - _t; _t = _n; } while (0)
#else
            long long *pt = nullptr;
            (void)pt;
#define FHQ(i) do {} while (0)
#endif
            for (int t = 0; t < T_; ++t) {
                const int par = t & 1;
                const int g = cl + t * A.ncl;
                const int b = g / A.Gb, gl = g - b * A.Gb;
                const int64_t s_in_batch = (int64_t)gl * TW + lane;
                FHQ(7);
                bar_wait(full, (uint32_t)(t & 1));
                FHQ(0);
                if (MODE == MODE_CH1D) ch1d_rhs<T>(slot, slot + TILE, kmax, lane, A.alpha);
                T v[Q];
#pragma unroll
                for (int k = 0; k < Q; ++k) v[k] = tld<T, LAY>(slot, k, lane);
                // the slot's reads are done (values in registers): hand it to the
                // async proxy for the next group's tile
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                if (lane == 0 && t + 1 < T_) issue(t + 1);
                FHQ(1);
                // ---- P1: zero-inflow forward sweep, carry, back-substitution functional
                {
                    T y0, y1, a0, a1, gs[4] = {T(0), T(0), T(0), T(0)};
                    if (kmax == Q) {
                        T hist[4] = {T(0), T(0), T(0), T(0)};
                        if (PER && spec_tile) {
                            p1_full<T, K, true>(v, cp, wp, y0, y1, a0, a1, hist);
#pragma unroll
                            for (int jx = 0; jx < 4; ++jx) {
                                const int64_t rr = A.srow[jx] - r0;
                                if (A.srow[jx] >= 0 && rr >= 0 && rr < Q) {
                                    const int j = (int)(rr & 3);
                                    gs[jx] = j == 0 ? hist[0] : j == 1 ? hist[1] : j == 2 ? hist[2] : hist[3];
                                }
                            }
                        } else {
                            p1_full<T, K, false>(v, cp, wp, y0, y1, a0, a1, hist);
                        }
                    } else if (PER && spec_tile) {
                        p1_sweep<T, K, true, false>(v, cp, wp, kmax, r0, A.srow, y0, y1, a0, a1, gs);
                    } else {
                        p1_sweep<T, K, false, false>(v, cp, wp, kmax, r0, A.srow, y0, y1, a0, a1, gs);
                    }
                    sm.rec[0][warp][lane][0] = y0;
                    sm.rec[0][warp][lane][1] = y1;
                    sm.rec[0][warp][lane][2] = a0;
                    sm.rec[0][warp][lane][3] = a1;
                    if (PER && spec_tile) {
#pragma unroll
                        for (int jx = 0; jx < 4; ++jx)
                            if (A.srow[jx] >= 0 && A.srow[jx] / Q == q) sm.spec[0][jx][lane] = gs[jx];
                    }
                    __syncwarp();
                    if (lane == 0) bar_arrive(&sm.p1done[par]);
                }
                FHQ(2);
                if (warp == 0) {
                    // the group's carry scan (cluster-wide), once every warp's P1 is in;
                    // the tile waits in shared memory meanwhile (the scan's registers)
#pragma unroll
                    for (int k = 0; k < Q; ++k) sm.park[k][lane] = v[k];
                    bar_wait(&sm.p1done[par], (uint32_t)((t >> 1) & 1));
                    FHQ(3);
                    hold_scan<T, K, PER, csmax<MODE>()>(A, sm, t, c, q0, nch, lane);
                    FHQ(4);
#pragma unroll
                    for (int k = 0; k < Q; ++k) v[k] = sm.park[k][lane];
                    __syncwarp();
                    if (lane == 0) bar_arrive(&sm.scandone[par]);
                }
                // ---- P2 on the same registers: inflows and x_l of the group, sweeps, x out
                bar_wait(&sm.scandone[par], (uint32_t)((t >> 1) & 1));
                FHQ(5);
                const T yi0 = sm.rec[0][warp][lane][0], yi1 = sm.rec[0][warp][lane][1];
                const T zi0 = sm.rec[0][warp][lane][2], zi1 = sm.rec[0][warp][lane][3];
                T xl0 = T(0), xl1 = T(0);
                if (PER) xl0 = sm.xl[0][lane][0], xl1 = sm.xl[0][lane][1];
                if (kmax == Q) p2_full<T, K, PER>(v, cp, yi0, yi1, zi0, zi1, xl0, xl1);
                else tile_solve<T, K, PER, false>(v, cp, kmax, yi0, yi1, zi0, zi1, xl0, xl1);
                if (PER && K == 2 && r0 + Q > A.n - 2) {
                    const int k2 = (int)(A.n - 2 - r0);
#pragma unroll
                    for (int k = 0; k < Q; ++k) {
                        if (k == k2) v[k] = xl0;
                        if (k == k2 + 1) v[k] = xl1;
                    }
                }
                FHQ(6);
                if (s_in_batch >= A.M) continue;
                if (LAY == LAY_CONTIG) {
                    // system = row of the output: 64 consecutive elements per lane
                    T *x = A.xout + (int64_t)b * A.bstride + s_in_batch * A.pitch + r0;
                    if (kmax == Q) {
#pragma unroll
                        for (int k = 0; k < Q; k += 16 / (int)sizeof(T)) {
                            if (sizeof(T) == 8)
                                __stcs(reinterpret_cast<double2 *>(x + k), make_double2((double)v[k], (double)v[k + 1]));
                            else
                                __stcs(reinterpret_cast<float4 *>(x + k),
                                       make_float4((float)v[k], (float)v[k + 1], (float)v[k + 2], (float)v[k + 3]));
                        }
                    } else {
#pragma unroll
                        for (int k = 0; k < Q; ++k)
                            if (k < kmax) __stcs(x + k, v[k]);
                    }
                } else {
                    // every row of the tile is one contiguous 32-system segment
                    int64_t Mo = A.pitch;
                    asm volatile("" : "+l"(Mo));
                    T *x = A.xout + (int64_t)b * A.bstride + r0 * Mo + s_in_batch;
#pragma unroll
                    for (int k = 0; k < Q; ++k) {
                        if (kmax == Q || k < kmax) __stcs(x, v[k]);
                        x += Mo;
                    }
                }
            }
#ifdef FH_PROF
            if (A.prof && lane == 0)
                for (int i = 0; i < 16; ++i) atomicAdd((unsigned long long *)&A.prof[warp * 16 + i], (unsigned long long)pacc[i]);
#endif
        }
    }
    // no CTA may leave while a peer can still write into its shared memory
    cg::this_cluster().sync();
}

}  // namespace fh
}  // namespace pb
