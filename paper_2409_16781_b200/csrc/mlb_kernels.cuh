// mlb_kernels.cuh - sm_100a device code of the D3Q19 time-step loop.
//
// One translation unit (mlb_api.cu includes this), compiled with
// -fmad=false: every floating-point operation below is a single IEEE
// rounding, in the operation order of the reference's canonical per-cell
// update (lb2d lattice.py:127-182 == kernels.py:199-245, generalised to 19
// velocities), so the populations this kernel writes are BIT-IDENTICAL to
// the CPU oracle's (oracle/d3q19_oracle.c, built with -ffp-contract=off).
// The update is a pure HBM-bound stencil (195 flop / 152 B in fp32): no
// tensor cores, the unfused multiplies cost nothing measurable.
//
// Velocity order (paper_2409_16781_b200/lattice.py): 0 rest; 1..4 = +x,+y,
// -x,-y; 5..8 = xy diagonals (the reference's D2Q9 order); 9,10 = +z,-z;
// 11..14 = (+x+z),(-x+z),(-x-z),(+x-z); 15..18 = (+y+z),(-y+z),(-y-z),(+y-z).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace mlb {

constexpr int Q = 19;

struct Geom {
    int nx, ny, nz;          // slab cells
    int zlo_src, zhi_src;    // storage planes that serve lz = -1 and lz = nz
    long long xp, plane, pop;  // row pitch, z-plane, population strides (elements)
};

template <typename T>
struct StepArgs {
    const T *__restrict__ fpre;
    T *__restrict__ fpost;
    const uint8_t *__restrict__ cls;
    Geom g;
    int z0;        // first slab plane this launch updates (blockIdx.z = 0)
    T omega;
    T k[Q];        // moving-wall terms 6 w_i (c_i . u_w), compute dtype
};

// class byte: low 3 bits = the reference's flag code (boundaries.py:20-24),
// bit 7 = "some neighbour is SOLID or MOVING_WALL" (cell needs the flag-test
// gather).  cls == 0 is a bulk fluid cell: 19 plain loads, no flag reads.
constexpr uint8_t CLS_FLAG = 0x07;
constexpr uint8_t CLS_NEAR_WALL = 0x80;

// ---------------------------------------------------------------------------
// collide: lattice.collide_cell (lattice.py:127-182) for 19 velocities.
// g is overwritten with the post-collision populations.
template <typename T>
__device__ __forceinline__ void collide(T (&g)[Q], const T omega)
{
    const T one = T(1.0), zero = T(0.0);
    const T c3 = T(3.0), c45 = T(4.5), c15 = T(1.5);
    const T w0 = T(1.0 / 3.0), ws = T(1.0 / 18.0), wd = T(1.0 / 36.0);

    const T rho = g[0] + g[1] + g[2] + g[3] + g[4] + g[5] + g[6] + g[7] + g[8]
                + g[9] + g[10] + g[11] + g[12] + g[13] + g[14] + g[15] + g[16]
                + g[17] + g[18];
    const T mx = g[1] - g[3] + g[5] - g[6] - g[7] + g[8] + g[11] - g[12] - g[13] + g[14];
    const T my = g[2] - g[4] + g[5] + g[6] - g[7] - g[8] + g[15] - g[16] - g[17] + g[18];
    const T mz = g[9] - g[10] + g[11] + g[12] - g[13] - g[14] + g[15] + g[16] - g[17] - g[18];
    T inv;
    if (rho != zero)
        inv = one / rho;
    else
        inv = zero;
    const T ux = mx * inv, uy = my * inv, uz = mz * inv;
    const T usq = ux * ux + uy * uy + uz * uz;
    const T um = one - c15 * usq;
    const T wr0 = w0 * rho, wrs = ws * rho, wrd = wd * rho;
    const T a = ux + uy, b = ux - uy, c = ux + uz, d = ux - uz, h = uy + uz,
            kk = uy - uz;

#define MLB_PAIR(cu, wr, ip, im)                                   \
    {                                                              \
        const T q_ = c45 * ((cu) * (cu));                          \
        const T t_ = c3 * (cu);                                    \
        const T p_ = um + q_;                                      \
        const T ep_ = (wr) * (p_ + t_);                            \
        const T em_ = (wr) * (p_ - t_);                            \
        g[ip] = g[ip] - omega * (g[ip] - ep_);                     \
        g[im] = g[im] - omega * (g[im] - em_);                     \
    }
    MLB_PAIR(ux, wrs, 1, 3)
    MLB_PAIR(uy, wrs, 2, 4)
    MLB_PAIR(a, wrd, 5, 7)
    MLB_PAIR(b, wrd, 8, 6)
    MLB_PAIR(uz, wrs, 9, 10)
    MLB_PAIR(c, wrd, 11, 13)
    MLB_PAIR(d, wrd, 14, 12)
    MLB_PAIR(h, wrd, 15, 17)
    MLB_PAIR(kk, wrd, 18, 16)
#undef MLB_PAIR
    {
        const T e0 = wr0 * um;
        g[0] = g[0] - omega * (g[0] - e0);
    }
}

// opposite direction, usable in constant expressions after unrolling
__host__ __device__ constexpr int opp(int i)
{
    return i == 0 ? 0
         : i <= 4 ? (i <= 2 ? i + 2 : i - 2)
         : i <= 8 ? (i <= 6 ? i + 2 : i - 2)
         : i == 9 ? 10 : i == 10 ? 9
         : i <= 14 ? (i <= 12 ? i + 2 : i - 2)
         : (i <= 16 ? i + 2 : i - 2);
}

// ---------------------------------------------------------------------------
// Fused pull-stream + bounce-back + BGK collide, one thread per cell
// (kernels.py:76-245 `cell`, :247-279 `fused`).  blockIdx = (x tile, y, plane).
// Reads fpre only, writes each FLUID cell of fpost once, nothing else.
template <typename T, int BX>
__global__ void __launch_bounds__(BX) step_kernel(const StepArgs<T> a)
{
    const Geom &gm = a.g;
    const int x = blockIdx.x * BX + threadIdx.x;
    if (x >= gm.nx)
        return;
    const int y = blockIdx.y;
    const int lz = a.z0 + blockIdx.z;

    // periodic wrap first, flag test second (kernels.py:83-96); y and z are
    // block-uniform, the x wrap touches only the two edge lanes of a row.
    const int xm = (x == 0) ? gm.nx - 1 : x - 1;          // source for c_x = +1
    const int xq = (x == gm.nx - 1) ? 0 : x + 1;          // source for c_x = -1
    const int ym = (y == 0) ? gm.ny - 1 : y - 1;
    const int yq = (y == gm.ny - 1) ? 0 : y + 1;
    const long long zc = (long long)(lz + 1) * gm.plane;
    const long long zm = (long long)((lz == 0) ? gm.zlo_src : lz) * gm.plane;
    const long long zq = (long long)((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) * gm.plane;
    const long long rc = (long long)y * gm.xp, rm = (long long)ym * gm.xp,
                    rq = (long long)yq * gm.xp;

    const long long d = zc + rc + x;
    const uint8_t cd = a.cls[d];
    if (cd & CLS_FLAG)
        return;  // non-fluid destination: never written (kernels.py:79-80)

    const T *__restrict__ f = a.fpre;
    const long long P = gm.pop;
    T g[Q];
    g[0] = f[d];

    if (cd == 0) {
#define MLB_PULL(i, zz, rr, xx) g[i] = f[(long long)(i) * P + (zz) + (rr) + (xx)];
        MLB_PULL(1, zc, rc, xm)  MLB_PULL(2, zc, rm, x)   MLB_PULL(3, zc, rc, xq)
        MLB_PULL(4, zc, rq, x)   MLB_PULL(5, zc, rm, xm)  MLB_PULL(6, zc, rm, xq)
        MLB_PULL(7, zc, rq, xq)  MLB_PULL(8, zc, rq, xm)  MLB_PULL(9, zm, rc, x)
        MLB_PULL(10, zq, rc, x)  MLB_PULL(11, zm, rc, xm) MLB_PULL(12, zm, rc, xq)
        MLB_PULL(13, zq, rc, xq) MLB_PULL(14, zq, rc, xm) MLB_PULL(15, zm, rm, x)
        MLB_PULL(16, zm, rq, x)  MLB_PULL(17, zq, rq, x)  MLB_PULL(18, zq, rm, x)
#undef MLB_PULL
    } else {
        // near a wall: SOLID source -> own opposite population, MOVING_WALL
        // source -> that plus the wall term, anything else (fluid, inlet,
        // outlet) -> plain pull (kernels.py:88-96, boundaries.py:10-12)
#define MLB_PULL(i, zz, rr, xx)                                         \
        {                                                               \
            const long long s_ = (zz) + (rr) + (xx);                    \
            const uint8_t m_ = a.cls[s_] & CLS_FLAG;                    \
            if (m_ == 1)                                                \
                g[i] = f[(long long)opp(i) * P + d];                    \
            else if (m_ == 2)                                           \
                g[i] = f[(long long)opp(i) * P + d] + a.k[i];           \
            else                                                        \
                g[i] = f[(long long)(i) * P + s_];                      \
        }
        MLB_PULL(1, zc, rc, xm)  MLB_PULL(2, zc, rm, x)   MLB_PULL(3, zc, rc, xq)
        MLB_PULL(4, zc, rq, x)   MLB_PULL(5, zc, rm, xm)  MLB_PULL(6, zc, rm, xq)
        MLB_PULL(7, zc, rq, xq)  MLB_PULL(8, zc, rq, xm)  MLB_PULL(9, zm, rc, x)
        MLB_PULL(10, zq, rc, x)  MLB_PULL(11, zm, rc, xm) MLB_PULL(12, zm, rc, xq)
        MLB_PULL(13, zq, rc, xq) MLB_PULL(14, zq, rc, xm) MLB_PULL(15, zm, rm, x)
        MLB_PULL(16, zm, rq, x)  MLB_PULL(17, zq, rq, x)  MLB_PULL(18, zq, rm, x)
#undef MLB_PULL
    }

    collide<T>(g, a.omega);

    T *__restrict__ o = a.fpost + d;
#pragma unroll
    for (int i = 0; i < Q; ++i)
        o[(long long)i * P] = g[i];
}

// ---------------------------------------------------------------------------
// Vectorised fused update: each thread owns a PACK of V = 16 / sizeof(T)
// consecutive cells in x (one 16-byte word per population), a warp covers
// LX packs in x by 32 / LX rows in y.  Per pack and population: one aligned
// 16-byte load; the ten populations with c_x = +-1 need the word shifted by
// one cell, which costs one extra scalar load of the element just outside
// the pack (an L1 hit: the neighbouring lane's word holds it).  Stores are
// aligned 16-byte words (pull scheme: destinations are never shifted).
//
// Walls stay branch-free: a warp whose packs are all bulk fluid takes the
// plain path; any other warp takes the "general" path as a whole, where a
// lane with wall links also loads its own cell's opposite populations and
// selects per cell and direction with the precomputed link masks
// (kernels.py:88-96: SOLID source -> own opposite population, MOVING_WALL
// source -> that plus the wall term).  No flag reads, no divergence.
template <typename T> struct Vec;
template <> struct Vec<float>  { using type = float4;  static constexpr int V = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int V = 2; };

template <typename T>
__device__ __forceinline__ void unpack(const typename Vec<T>::type &v, T (&o)[Vec<T>::V]);
template <>
__device__ __forceinline__ void unpack<float>(const float4 &v, float (&o)[4])
{ o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
template <>
__device__ __forceinline__ void unpack<double>(const double2 &v, double (&o)[2])
{ o[0] = v.x; o[1] = v.y; }

__device__ __forceinline__ float4 pack(const float (&o)[4]) { return make_float4(o[0], o[1], o[2], o[3]); }
__device__ __forceinline__ double2 pack(const double (&o)[2]) { return make_double2(o[0], o[1]); }

// The V values pulled along a direction with x component CX from the row
// starting at `row` (already offset to population, plane and row).
template <typename T, int CX>
__device__ __forceinline__ void pull_pack(const T *__restrict__ row, int x0, int xl, int xr,
                                          T (&o)[Vec<T>::V])
{
    constexpr int V = Vec<T>::V;
    using VT = typename Vec<T>::type;
    T w[V];
    unpack<T>(*reinterpret_cast<const VT *>(row + x0), w);
    if (CX == 0) {
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = w[j];
    } else if (CX > 0) {  // source x - 1
        o[0] = row[xl];
#pragma unroll
        for (int j = 1; j < V; ++j) o[j] = w[j - 1];
    } else {              // source x + 1
#pragma unroll
        for (int j = 0; j < V - 1; ++j) o[j] = w[j + 1];
        o[V - 1] = row[xr];
    }
}

// direction table: X(i, c_x, plane offset, row offset)
#define MLB_DIRS(X)                                                              \
    X(1, 1, zc, rc)   X(2, 0, zc, rm)   X(3, -1, zc, rc)  X(4, 0, zc, rq)        \
    X(5, 1, zc, rm)   X(6, -1, zc, rm)  X(7, -1, zc, rq)  X(8, 1, zc, rq)        \
    X(9, 0, zm, rc)   X(10, 0, zq, rc)  X(11, 1, zm, rc)  X(12, -1, zm, rc)      \
    X(13, -1, zq, rc) X(14, 1, zq, rc)  X(15, 0, zm, rm)  X(16, 0, zm, rq)       \
    X(17, 0, zq, rq)  X(18, 0, zq, rm)

template <typename T, int LX>
__global__ void __launch_bounds__(128)
step_vec_kernel(const StepArgs<T> a, const unsigned long long *__restrict__ links)
{
    constexpr int V = Vec<T>::V;
    using VT = typename Vec<T>::type;
    constexpr int RPW = 32 / LX;        // rows per warp
    constexpr unsigned FULL = 0xffffffffu;
    const Geom &gm = a.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * LX + (lane % LX)) * V;
    const int y = blockIdx.y * (4 * RPW) + warp * RPW + lane / LX;
    const int lz = a.z0 + blockIdx.z;
    const bool inrange = (x0 < gm.nx) && (y < gm.ny);

    const long long zc = (long long)(lz + 1) * gm.plane;
    const long long zm = (long long)((lz == 0) ? gm.zlo_src : lz) * gm.plane;
    const long long zq = (long long)((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) * gm.plane;
    const int yy = inrange ? y : 0;
    const int ym = (yy == 0) ? gm.ny - 1 : yy - 1;
    const int yq = (yy == gm.ny - 1) ? 0 : yy + 1;
    const long long rc = (long long)yy * gm.xp, rm = (long long)ym * gm.xp,
                    rq = (long long)yq * gm.xp;
    const int xx = inrange ? x0 : 0;
    const int xl = (xx == 0) ? gm.nx - 1 : xx - 1;
    const int xr = (xx + V >= gm.nx) ? 0 : xx + V;
    const long long d = zc + rc + xx;

    // class bytes of the pack, one 16/32-bit word
    unsigned c4;
    if (V == 4)
        c4 = *reinterpret_cast<const unsigned *>(a.cls + d);
    else
        c4 = *reinterpret_cast<const unsigned short *>(a.cls + d);
    if (!inrange)
        c4 = (V == 4) ? 0x01010101u : 0x0101u;  // nothing to do here
    bool fluid[V];
    bool anyfluid = false, allfluid = true;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        fluid[j] = ((c4 >> (8 * j)) & CLS_FLAG) == 0;
        anyfluid |= fluid[j];
        allfluid &= fluid[j];
    }
    const bool bulk = (c4 == 0);
    const bool general = !__all_sync(FULL, bulk || !anyfluid);  // warp-uniform
    if (!anyfluid)
        return;

    const T *__restrict__ f = a.fpre;
    const long long P = gm.pop;
    T g[Q][V];
    unpack<T>(*reinterpret_cast<const VT *>(f + d), g[0]);

    if (!general) {
#define MLB_X(i, CX, Z, R) pull_pack<T, CX>(f + (long long)(i) * P + (Z) + (R), xx, xl, xr, g[i]);
        MLB_DIRS(MLB_X)
#undef MLB_X
    } else {
        // link masks of the pack (zero for bulk cells; garbage-free for
        // non-fluid ones, which are never stored)
        unsigned lo[V], hi[V];
#pragma unroll
        for (int j = 0; j < V; ++j) { lo[j] = 0u; hi[j] = 0u; }
        if (!bulk) {
#pragma unroll
            for (int j = 0; j < V; j += 2) {
                const ulonglong2 m = *reinterpret_cast<const ulonglong2 *>(links + d + j);
                lo[j] = (unsigned)m.x;     hi[j] = (unsigned)(m.x >> 32);
                lo[j + 1] = (unsigned)m.y; hi[j + 1] = (unsigned)(m.y >> 32);
            }
        }
        unsigned anylo = 0u;
#pragma unroll
        for (int j = 0; j < V; ++j) anylo |= lo[j];
#define MLB_X(i, CX, Z, R)                                                        \
        {                                                                         \
            pull_pack<T, CX>(f + (long long)(i) * P + (Z) + (R), xx, xl, xr, g[i]); \
            if (anylo & (1u << (i))) {                                            \
                T c_[V];                                                          \
                unpack<T>(*reinterpret_cast<const VT *>(f + (long long)opp(i) * P + d), c_); \
                _Pragma("unroll")                                                 \
                for (int j = 0; j < V; ++j) {                                     \
                    if (lo[j] & (1u << (i)))                                      \
                        g[i][j] = (hi[j] & (1u << (i))) ? c_[j] + a.k[i] : c_[j]; \
                }                                                                 \
            }                                                                     \
        }
        MLB_DIRS(MLB_X)
#undef MLB_X
    }

    // collide each cell of the pack (lattice.collide_cell order)
#pragma unroll
    for (int j = 0; j < V; ++j) {
        T gc[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) gc[i] = g[i][j];
        collide<T>(gc, a.omega);
#pragma unroll
        for (int i = 0; i < Q; ++i) g[i][j] = gc[i];
    }

    T *__restrict__ o = a.fpost + d;
    if (allfluid) {
#pragma unroll
        for (int i = 0; i < Q; ++i)
            *reinterpret_cast<VT *>(o + (long long)i * P) = pack(g[i]);
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j)
            if (fluid[j]) {
#pragma unroll
                for (int i = 0; i < Q; ++i)
                    o[(long long)i * P + j] = g[i][j];
            }
    }
}

// ---------------------------------------------------------------------------
// Class table and link masks from the padded flag block (halo planes already
// filled).  One thread per padded element of storage planes [0, nz+2).
//   links[d] bit i      (1 <= i <= 18): the source cell of direction i is a
//                        wall (SOLID or MOVING_WALL) -> bounce-back link
//   links[d] bit 32 + i: that wall is a MOVING_WALL -> add the wall term k_i
// Direction i's source is the neighbour at -c_i, with the same periodic
// wrap / halo-plane rule as the step kernels.
__device__ __forceinline__ constexpr int dir_index(int cx, int cy, int cz)
{
    // inverse of the velocity table in lattice.py; -1 for the 8 corners / rest
    if (cz == 0) {
        if (cy == 0) return cx == 1 ? 1 : cx == -1 ? 3 : 0;
        if (cx == 0) return cy == 1 ? 2 : 4;
        return cy == 1 ? (cx == 1 ? 5 : 6) : (cx == -1 ? 7 : 8);
    }
    if (cx == 0 && cy == 0) return cz == 1 ? 9 : 10;
    if (cy == 0) return cz == 1 ? (cx == 1 ? 11 : 12) : (cx == -1 ? 13 : 14);
    if (cx == 0) return cz == 1 ? (cy == 1 ? 15 : 16) : (cy == -1 ? 17 : 18);
    return -1;
}

__global__ void build_cls_kernel(const uint8_t *__restrict__ flags,
                                 uint8_t *__restrict__ cls,
                                 unsigned long long *__restrict__ links, const Geom gm)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= gm.xp)
        return;
    const int y = blockIdx.y;
    const int sz = blockIdx.z;  // storage plane
    const long long d = (long long)sz * gm.plane + (long long)y * gm.xp + x;
    if (x >= gm.nx) {
        cls[d] = 1;  // row padding: solid, never written
        links[d] = 0ull;
        return;
    }
    const uint8_t fl = flags[d];
    if (sz == 0 || sz == gm.nz + 1) {
        cls[d] = fl;  // halo planes are only ever sources
        links[d] = 0ull;
        return;
    }
    const int lz = sz - 1;
    // index 0: same, 1: the "minus" neighbour (source for c = +1), 2: the "plus" one
    const int xs[3] = {x, (x == 0) ? gm.nx - 1 : x - 1, (x == gm.nx - 1) ? 0 : x + 1};
    const int ys[3] = {y, (y == 0) ? gm.ny - 1 : y - 1, (y == gm.ny - 1) ? 0 : y + 1};
    const int zs[3] = {sz, (lz == 0) ? gm.zlo_src : lz, (lz == gm.nz - 1) ? gm.zhi_src : lz + 2};
    const int cof[3] = {0, 1, -1};  // the c component served by index 0/1/2
    unsigned long long lk = 0ull;
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                const int i = dir_index(cof[dx], cof[dy], cof[dz]);
                if (i <= 0)
                    continue;  // rest particle / the 8 corners: no D3Q19 link
                const uint8_t m = flags[(long long)zs[dz] * gm.plane
                                        + (long long)ys[dy] * gm.xp + xs[dx]];
                if (m == 1 || m == 2)
                    lk |= 1ull << i;
                if (m == 2)
                    lk |= 1ull << (32 + i);
            }
    cls[d] = fl | (lk ? CLS_NEAR_WALL : 0);
    links[d] = (fl == 0) ? lk : 0ull;
}

// ---------------------------------------------------------------------------
// Open-boundary pass (engine.py:156-180), driven by index lists.
template <typename T>
struct InletVals { T v[Q]; };

template <typename T>
__global__ void inlet_kernel(T *__restrict__ f, const long long *__restrict__ idx,
                             long long n, long long pop, const InletVals<T> vals)
{
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n)
        return;
    const long long d = idx[j];
#pragma unroll
    for (int i = 0; i < Q; ++i)
        f[(long long)i * pop + d] = vals.v[i];
}

// mode 0: f[d] <- f[d-1] directly (no outlet cell is another's source)
// mode 1: tmp[i][j] <- f[d-1]        mode 2: f[d] <- tmp[i][j]
template <typename T>
__global__ void outlet_kernel(T *__restrict__ f, T *__restrict__ tmp,
                              const long long *__restrict__ idx, long long n,
                              long long pop, long long tmp_stride, int mode)
{
    const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n)
        return;
    const long long d = idx[j];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        if (mode == 0)
            f[(long long)i * pop + d] = f[(long long)i * pop + d - 1];
        else if (mode == 1)
            tmp[(long long)i * tmp_stride + j] = f[(long long)i * pop + d - 1];
        else
            f[(long long)i * pop + d] = tmp[(long long)i * tmp_stride + j];
    }
}

// ---------------------------------------------------------------------------
// Halo copy: 5 crossing populations of one boundary plane, 16-byte words.
struct HaloArgs {
    long long dst_off[5];  // element offsets of the 5 destination planes
    long long src_off[5];
    long long words;       // 16-byte words per plane
};

__global__ void halo_copy_kernel(const void *__restrict__ src, void *__restrict__ dst,
                                 const HaloArgs h, int itemsize)
{
    const long long w = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (w >= h.words)
        return;
    const int q = blockIdx.y;
    const uint4 *s = reinterpret_cast<const uint4 *>(
        static_cast<const char *>(src) + h.src_off[q] * itemsize);
    uint4 *d = reinterpret_cast<uint4 *>(static_cast<char *>(dst) + h.dst_off[q] * itemsize);
    d[w] = s[w];
}

// ---------------------------------------------------------------------------
// Macroscopic fields (engine.py:104-118): float64, all cells, true division.
template <typename T>
__device__ __forceinline__ void cell_moments(const T *__restrict__ f, long long d,
                                             long long pop, double &r, double &mx,
                                             double &my, double &mz, int *bad)
{
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        v[i] = (double)f[(long long)i * pop + d];
        if (bad && !isfinite(v[i]))
            ++*bad;
    }
    r = v[0];
#pragma unroll
    for (int i = 1; i < Q; ++i)
        r = r + v[i];
    mx = v[1] - v[3] + v[5] - v[6] - v[7] + v[8] + v[11] - v[12] - v[13] + v[14];
    my = v[2] - v[4] + v[5] + v[6] - v[7] - v[8] + v[15] - v[16] - v[17] + v[18];
    mz = v[9] - v[10] + v[11] + v[12] - v[13] - v[14] + v[15] + v[16] - v[17] - v[18];
}

template <typename T>
__global__ void macro_kernel(const T *__restrict__ f, const Geom gm,
                             double *__restrict__ rho, double *__restrict__ ux,
                             double *__restrict__ uy, double *__restrict__ uz)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= gm.nx)
        return;
    const int y = blockIdx.y, lz = blockIdx.z;
    const long long d = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp + x;
    const long long o = ((long long)lz * gm.ny + y) * gm.nx + x;
    double r, mx, my, mz;
    cell_moments<T>(f, d, gm.pop, r, mx, my, mz, nullptr);
    rho[o] = r;
    ux[o] = (r != 0.0) ? mx / r : 0.0;
    uy[o] = (r != 0.0) ? my / r : 0.0;
    uz[o] = (r != 0.0) ? mz / r : 0.0;
}

template <typename T>
__global__ void probe_kernel(const T *__restrict__ f, const Geom gm, int x, int y,
                             int lz, double *__restrict__ out4)
{
    const long long d = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp + x;
    double r, mx, my, mz;
    cell_moments<T>(f, d, gm.pop, r, mx, my, mz, nullptr);
    out4[0] = r;
    out4[1] = (r != 0.0) ? mx / r : 0.0;
    out4[2] = (r != 0.0) ? my / r : 0.0;
    out4[3] = (r != 0.0) ? mz / r : 0.0;
}

// ---------------------------------------------------------------------------
// Scalar diagnostics: per-thread accumulation over a fixed row assignment,
// warp-shuffle tree, fixed-order cross-warp sum, per-block partials, then a
// single-block final pass.  No float atomics: bitwise reproducible.
constexpr int DIAG_N = 8;        // mass, px, py, pz, ke, max|u|, nonfinite, fluid cells
constexpr int DIAG_THREADS = 256;

__device__ __forceinline__ void diag_combine(double (&a)[DIAG_N], const double (&b)[DIAG_N])
{
#pragma unroll
    for (int i = 0; i < DIAG_N; ++i)
        a[i] = (i == 5) ? fmax(a[i], b[i]) : a[i] + b[i];
}

__device__ __forceinline__ void diag_block_reduce(double (&acc)[DIAG_N], double *out)
{
    __shared__ double sm[DIAG_THREADS / 32][DIAG_N];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        double o[DIAG_N];
#pragma unroll
        for (int i = 0; i < DIAG_N; ++i)
            o[i] = __shfl_down_sync(0xffffffffu, acc[i], off);
        diag_combine(acc, o);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < DIAG_N; ++i)
            sm[warp][i] = acc[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[DIAG_N];
#pragma unroll
        for (int i = 0; i < DIAG_N; ++i)
            t[i] = sm[0][i];
        for (int w = 1; w < DIAG_THREADS / 32; ++w)
            diag_combine(t, sm[w]);
#pragma unroll
        for (int i = 0; i < DIAG_N; ++i)
            out[i] = t[i];
    }
}

template <typename T>
__global__ void __launch_bounds__(DIAG_THREADS)
diag_kernel(const T *__restrict__ f, const uint8_t *__restrict__ cls, const Geom gm,
            double *__restrict__ partials)
{
    double acc[DIAG_N];
#pragma unroll
    for (int i = 0; i < DIAG_N; ++i)
        acc[i] = 0.0;
    const long long rows = (long long)gm.nz * gm.ny;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
        const int lz = (int)(r / gm.ny), y = (int)(r % gm.ny);
        const long long base = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp;
        for (int x = threadIdx.x; x < gm.nx; x += DIAG_THREADS) {
            const long long d = base + x;
            double rr, mx, my, mz;
            int bad = 0;
            cell_moments<T>(f, d, gm.pop, rr, mx, my, mz, &bad);
            acc[0] += rr;
            acc[6] += (double)bad;
            if ((cls[d] & CLS_FLAG) == 0) {
                acc[7] += 1.0;
                acc[1] += mx;
                acc[2] += my;
                acc[3] += mz;
                if (rr != 0.0) {
                    const double u2 = (mx * mx + my * my + mz * mz) / (rr * rr);
                    acc[4] += 0.5 * rr * u2;
                    acc[5] = fmax(acc[5], sqrt(u2));
                }
            }
        }
    }
    diag_block_reduce(acc, partials + (long long)blockIdx.x * DIAG_N);
}

__global__ void __launch_bounds__(DIAG_THREADS)
diag_final_kernel(const double *__restrict__ partials, int nblocks,
                  double *__restrict__ out)
{
    double acc[DIAG_N];
#pragma unroll
    for (int i = 0; i < DIAG_N; ++i)
        acc[i] = 0.0;
    for (int b = threadIdx.x; b < nblocks; b += DIAG_THREADS) {
        double p[DIAG_N];
#pragma unroll
        for (int i = 0; i < DIAG_N; ++i)
            p[i] = partials[(long long)b * DIAG_N + i];
        diag_combine(acc, p);
    }
    diag_block_reduce(acc, out);
}

}  // namespace mlb
