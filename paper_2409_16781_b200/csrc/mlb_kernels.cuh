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
// Class table from the padded flag block (halo planes already filled).
// One thread per padded element of storage planes [0, nz+2).
__global__ void build_cls_kernel(const uint8_t *__restrict__ flags,
                                 uint8_t *__restrict__ cls, const Geom gm)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= gm.xp)
        return;
    const int y = blockIdx.y;
    const int sz = blockIdx.z;  // storage plane
    const long long d = (long long)sz * gm.plane + (long long)y * gm.xp + x;
    if (x >= gm.nx) {
        cls[d] = 1;  // row padding: solid, never written
        return;
    }
    const uint8_t fl = flags[d];
    if (sz == 0 || sz == gm.nz + 1) {
        cls[d] = fl;  // halo planes are only ever sources
        return;
    }
    const int lz = sz - 1;
    const int xs[3] = {x, (x == 0) ? gm.nx - 1 : x - 1, (x == gm.nx - 1) ? 0 : x + 1};
    const int ys[3] = {y, (y == 0) ? gm.ny - 1 : y - 1, (y == gm.ny - 1) ? 0 : y + 1};
    const int zs[3] = {sz, (lz == 0) ? gm.zlo_src : lz, (lz == gm.nz - 1) ? gm.zhi_src : lz + 2};
    bool wall = false;
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
            for (int dx = 0; dx < 3; ++dx) {
                const int nnz = (dx != 0) + (dy != 0) + (dz != 0);
                if (nnz == 0 || nnz == 3)
                    continue;  // D3Q19 has no corner links
                const uint8_t m = flags[(long long)zs[dz] * gm.plane
                                        + (long long)ys[dy] * gm.xp + xs[dx]];
                wall |= (m == 1) || (m == 2);
            }
    cls[d] = fl | (wall ? CLS_NEAR_WALL : 0);
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
