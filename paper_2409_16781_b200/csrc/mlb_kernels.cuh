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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

namespace mlb {

constexpr int Q = 19;

// Storage type TS -> compute type and the two conversions.  float and double
// compute in their own type; __half is the reference's MIXED1 mode
// (fields.py:24): stored as binary16, upcast exactly on load, computed in
// float, rounded to nearest even on store (kernels.py:435-455).
template <typename TS> struct Store;
template <> struct Store<float> {
    using C = float;
    static __host__ __device__ __forceinline__ float up(float v) { return v; }
    static __host__ __device__ __forceinline__ float down(float v) { return v; }
};
template <> struct Store<double> {
    using C = double;
    static __host__ __device__ __forceinline__ double up(double v) { return v; }
    static __host__ __device__ __forceinline__ double down(double v) { return v; }
};
// MIXED2 (fields.py:25): float in memory, double arithmetic.  The element type
// is a 4-byte wrapper so that the templates can tell it from plain float.
struct f32w { float v; };
template <> struct Store<f32w> {
    using C = double;
    static __host__ __device__ __forceinline__ double up(f32w x) { return (double)x.v; }
    static __host__ __device__ __forceinline__ f32w down(double v) { f32w r; r.v = (float)v; return r; }
};
template <> struct Store<__half> {
    using C = float;
    static __host__ __device__ __forceinline__ float up(__half v) { return __half2float(v); }
    static __host__ __device__ __forceinline__ __half down(float v) { return __float2half_rn(v); }
};

struct Geom {
    int nx, ny, nz;          // slab cells
    int zlo_src, zhi_src;    // storage planes that serve lz = -1 and lz = nz
    long long xp, plane, pop;  // row pitch, z-plane, population strides (elements)
};

// Per-cell class word, computed from the flags (cell_class, inside build_kind_kernel):
//   bits 0..2   the reference's flag code (boundaries.py:20-24)
//   bit  2 + i  (i = 1..18) the source cell of direction i is a wall (SOLID or
//               MOVING_WALL): that link bounces back
//   bit  31     some bouncing link hits a MOVING_WALL: mlinks[d] bit i says which
// cls == 0 is a bulk fluid cell.  One 4-byte load per cell tells the kernel
// everything the reference learns from 19 flag reads (kernels.py:76-197).
constexpr uint32_t CLS_FLAG = 0x7u;
constexpr uint32_t CLS_MOVING = 0x80000000u;
__host__ __device__ constexpr uint32_t cls_link(int i) { return 1u << (2 + i); }

// What the kernels actually read per cell is ONE BYTE: `kind[d]`, an index into
// a per-plan dictionary `tab` of the distinct (class word, moving-wall link bits)
// pairs of the geometry (build_kind_kernel).  Index 0 is the bulk fluid cell
// (class word 0): a pack of cells whose kind bytes are all zero needs nothing
// else.  Everything else - walls, inlet / outlet cells, fluid cells next to a
// wall - looks its pair up in the table (at most 2 KB, L1-resident).  A cavity
// has ~30 distinct pairs; a geometry with more than 254 uses the escape index
// 255 for the overflow cells, which read the full-width arrays `cls_full` /
// `ml_full` (kept only in that case).  Compared with a 4-byte class word per
// cell this takes 3 B per update off the HBM traffic (2 % in fp32, 4 % with
// fp16 storage) and 7 B per cell off the footprint.
constexpr uint32_t KIND_ESCAPE = 255u;
struct ClsTab {
    const uint8_t *__restrict__ kind;
    const uint2 *__restrict__ tab;          // [256]: x = class word, y = moving-wall link bits
    const uint32_t *__restrict__ cls_full;  // escape cells only (may be NULL)
    const uint32_t *__restrict__ ml_full;
};
__device__ __forceinline__ uint32_t cls_of(const ClsTab &t, uint32_t k, int d)
{
    return k == KIND_ESCAPE ? t.cls_full[d] : __ldg(&t.tab[k].x);
}
__device__ __forceinline__ uint32_t mlinks_of(const ClsTab &t, uint32_t k, int d)
{
    return k == KIND_ESCAPE ? t.ml_full[d] : __ldg(&t.tab[k].y);
}

template <typename TS>
struct StepArgs {
    using T = typename Store<TS>::C;  // compute type
    // one base pointer per population (host-computed: keeps the 64-bit
    // q * pop products out of the kernel; an address is then a single
    // IMAD.WIDE of a 32-bit in-population offset onto a constant-bank base)
    const TS *pre[Q];
    TS *post[Q];
    ClsTab ct;     // per-cell kind byte + dictionary of class words, see below
    Geom g;
    int z0;        // first slab plane this launch updates (blockIdx.z = 0)
    int passthrough;  // 1: non-fluid cells are rewritten with fpre's value (see step_cell)
    int fuse_open;    // 1 (pack kernels, pass-through only): apply the open-boundary pass
                      // (engine.py:156-180) to the cells of the pack before storing
    int pf_dz, pf_dy; // pack kernels: L2-prefetch the lines of the cells pf_dz planes + pf_dy
                      // rows ahead (both 0 = off), see prefetch_ahead
    int pf_bulk;      // 1: as bulk row prefetches (prefetch_rows), 0: one lane per line
    TS inlet[Q];      // equilibrium(1, u_in, 0, 0), storage dtype
    T omega;
    T k[Q];        // moving-wall terms 6 w_i (c_i . u_w), compute dtype
    unsigned int *work;   // staged kernel: the launch's work counter (zeroed by the host)
};

// Fused halo exchange (z-slabs over peer memory).  The launch
// that updates a slab's boundary plane also stores the 5 populations that
// cross that face straight into the ring neighbour's halo plane - a pointer
// into the neighbour GPU's population block, mapped over NVLink (CUDA IPC /
// peer access): plane lz = nz-1, c_z = +1 set -> `hi[j]`, the start of
// population UP[j]'s halo plane lz = -1 of the slab above; plane lz = 0,
// c_z = -1 set -> `lo[j]`, population DOWN[j]'s halo plane lz = nz of the slab
// below.  The halo planes have the row pitch of this slab (same nx, ny,
// dtype).  A NULL first pointer disables that face.  The values and the set
// of cells stored are exactly those of the local store, so the neighbour's
// halo ends up byte-identical to a copy of the plane after the launch.
__host__ __device__ constexpr int halo_up(int j)    // c_z = +1: 9, 11, 12, 15, 16
{ return j == 0 ? 9 : j == 1 ? 11 : j == 2 ? 12 : j == 3 ? 15 : 16; }
__host__ __device__ constexpr int halo_down(int j)  // c_z = -1: 10, 13, 14, 17, 18
{ return j == 0 ? 10 : j == 1 ? 13 : j == 2 ? 14 : j == 3 ? 17 : 18; }
template <typename TS>
struct PushArgs {
    TS *lo[5];
    TS *hi[5];
};

// ---------------------------------------------------------------------------
// Lane algebra: the collide below is written once over a "lane" type L.
//   float, double : one cell, plain IEEE operators;
//   float2        : TWO cells side by side on Blackwell's packed-fp32
//                   instructions (FADD2 / FMUL2 / FFMA2, sm_100+): each is one
//                   issue slot for two independent round-to-nearest results.
//                   a - b is FFMA2(b, -1, a): the product is exact, the sum is
//                   rounded once - bit-identical to the scalar subtraction.
//                   ptxas contracts a packed multiply followed by a packed ADD
//                   (see addm below), so the packed collide writes its sums
//                   of products as differences of the exactly negated product
//                   (um + 4.5 cu^2 = um - (-4.5) cu^2); only 3 sums per cell
//                   stay scalar, and a cell's 195 unfused operations cost
//                   ~100 issue slots instead of 195.
// Every element of every result is the same correctly rounded value the
// scalar code (and the CPU oracle) produces.
template <typename L> struct Alg;
template <> struct Alg<float> {
    using S = float;
    static constexpr bool packed = false;
    static __device__ __forceinline__ float cst(float v) { return v; }
    static __device__ __forceinline__ float add(float a, float b) { return a + b; }
    static __device__ __forceinline__ float sub(float a, float b) { return a - b; }
    static __device__ __forceinline__ float mul(float a, float b) { return a * b; }
    static __device__ __forceinline__ float addm(float a, float m) { return a + m; }
    static __device__ __forceinline__ float subm(float a, float m) { return a - m; }
    static __device__ __forceinline__ float rcp0(float r) { return r != 0.0f ? 1.0f / r : 0.0f; }
};
template <> struct Alg<double> {
    using S = double;
    static constexpr bool packed = false;
    static __device__ __forceinline__ double cst(double v) { return v; }
    static __device__ __forceinline__ double add(double a, double b) { return a + b; }
    static __device__ __forceinline__ double sub(double a, double b) { return a - b; }
    static __device__ __forceinline__ double mul(double a, double b) { return a * b; }
    static __device__ __forceinline__ double addm(double a, double m) { return a + m; }
    static __device__ __forceinline__ double subm(double a, double m) { return a - m; }
    static __device__ __forceinline__ double rcp0(double r) { return r != 0.0 ? 1.0 / r : 0.0; }
};
template <> struct Alg<float2> {
    using S = float;
#ifdef MLB_SCALAR_SUMS   // A/B builds only: every sum that consumes a product per element
    static constexpr bool packed = false;
#else
    static constexpr bool packed = true;
#endif
    static __device__ __forceinline__ float2 cst(float v) { return make_float2(v, v); }
    static __device__ __forceinline__ float2 add(float2 a, float2 b) { return __fadd2_rn(a, b); }
    static __device__ __forceinline__ float2 sub(float2 a, float2 b)
    { return __ffma2_rn(b, make_float2(-1.0f, -1.0f), a); }
    static __device__ __forceinline__ float2 mul(float2 a, float2 b) { return __fmul2_rn(a, b); }
    // a + m / a - m where m is the result of a mul().  ptxas 12.9 contracts a
    // packed multiply followed by a packed add into FFMA2 - even for
    // mul.rn.f32x2 + add.rn.f32x2 in PTX, even with --fmad=false - which
    // skips the product's rounding (found as a 1-half-ulp parity failure, once
    // in ~20 000 values).  Scalar adds are not contracted (-fmad=false holds
    // for them), so the few true sums of a product are done per element.
    // The DIFFERENCE a - m is safe as FFMA2(m, -1, a) (exact product, one
    // rounding; ptxas leaves that form alone - FFMA2(m, +1, a) it rewrites to
    // an add and then contracts).  So the packed collide turns its sums of
    // products into differences of the exactly negated product (a + c*x =
    // a - (-c)*x, same bits: rounding to nearest is symmetric), see collide.
    static __device__ __forceinline__ float2 addm(float2 a, float2 m)
    { return make_float2(a.x + m.x, a.y + m.y); }
    static __device__ __forceinline__ float2 subm(float2 a, float2 m)
#ifdef MLB_SCALAR_SUMS
    { return make_float2(a.x - m.x, a.y - m.y); }
#else
    { return __ffma2_rn(m, make_float2(-1.0f, -1.0f), a); }
#endif
    static __device__ __forceinline__ float2 rcp0(float2 r)
    { return make_float2(r.x != 0.0f ? 1.0f / r.x : 0.0f, r.y != 0.0f ? 1.0f / r.y : 0.0f); }
};

// collide: lattice.collide_cell (lattice.py:127-182) for 19 velocities, same
// operation order.  g is overwritten with the post-collision populations.
template <typename L>
__device__ __forceinline__ void collide(L (&g)[Q], const typename Alg<L>::S omega_)
{
    using A = Alg<L>;
    using S = typename A::S;
    const L one = A::cst(S(1.0)), omega = A::cst(omega_);
    const L c3 = A::cst(S(3.0)), c45 = A::cst(S(4.5)), c15 = A::cst(S(1.5));
    const L w0 = A::cst(S(1.0 / 3.0)), ws = A::cst(S(1.0 / 18.0)), wd = A::cst(S(1.0 / 36.0));

    L rho = A::add(g[0], g[1]);
#pragma unroll
    for (int i = 2; i < Q; ++i)
        rho = A::add(rho, g[i]);
    // mx = g1 - g3 + g5 - g6 - g7 + g8 + g11 - g12 - g13 + g14, left to right
    const L mx = A::add(A::sub(A::sub(A::add(A::add(A::sub(A::sub(A::add(A::sub(
        g[1], g[3]), g[5]), g[6]), g[7]), g[8]), g[11]), g[12]), g[13]), g[14]);
    // my = g2 - g4 + g5 + g6 - g7 - g8 + g15 - g16 - g17 + g18
    const L my = A::add(A::sub(A::sub(A::add(A::sub(A::sub(A::add(A::add(A::sub(
        g[2], g[4]), g[5]), g[6]), g[7]), g[8]), g[15]), g[16]), g[17]), g[18]);
    // mz = g9 - g10 + g11 + g12 - g13 - g14 + g15 + g16 - g17 - g18
    const L mz = A::sub(A::sub(A::add(A::add(A::sub(A::sub(A::add(A::add(A::sub(
        g[9], g[10]), g[11]), g[12]), g[13]), g[14]), g[15]), g[16]), g[17]), g[18]);
    const L inv = A::rcp0(rho);  // rho != 0 ? 1 / rho : 0
    const L ux = A::mul(mx, inv), uy = A::mul(my, inv), uz = A::mul(mz, inv);
    // (addm / subm: a sum one of whose operands is a product, see Alg<float2>)
    const L usq = A::addm(A::addm(A::mul(ux, ux), A::mul(uy, uy)), A::mul(uz, uz));
    // (packed lanes: per element, so that every FFMA2 in the library keeps the one
    // checkable form (m, -1, a) - ptxas would write this one as (m, -R, 1))
    L um;
    if constexpr (A::packed) um = A::addm(one, A::mul(A::cst(S(-1.5)), usq));
    else um = A::subm(one, A::mul(c15, usq));
    const L wr0 = A::mul(w0, rho), wrs = A::mul(ws, rho), wrd = A::mul(wd, rho);
    const L a = A::add(ux, uy), b = A::sub(ux, uy), c = A::add(ux, uz), d = A::sub(ux, uz),
            h = A::add(uy, uz), kk = A::sub(uy, uz);

    // packed lanes: um + 4.5 cu^2 and p + 3 cu as differences of the negated
    // products (see Alg<float2>::subm) - same values, bit for bit
    const L nc3 = A::cst(S(-3.0)), nc45 = A::cst(S(-4.5));
#define MLB_PAIR(cu, wr, ip, im)                                               \
    {                                                                          \
        const L t_ = A::mul(c3, (cu));                                         \
        L p_, ep_;                                                             \
        if constexpr (A::packed) {                                             \
            p_ = A::subm(um, A::mul(nc45, A::mul((cu), (cu))));                \
            ep_ = A::mul((wr), A::subm(p_, A::mul(nc3, (cu))));                \
        } else {                                                               \
            p_ = A::addm(um, A::mul(c45, A::mul((cu), (cu))));                 \
            ep_ = A::mul((wr), A::addm(p_, t_));                               \
        }                                                                      \
        const L em_ = A::mul((wr), A::subm(p_, t_));                           \
        g[ip] = A::subm(g[ip], A::mul(omega, A::subm(g[ip], ep_)));            \
        g[im] = A::subm(g[im], A::mul(omega, A::subm(g[im], em_)));            \
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
        const L e0 = A::mul(wr0, um);
        g[0] = A::subm(g[0], A::mul(omega, A::subm(g[0], e0)));
    }
}

// collide V cells held as g[direction][cell], one by one ...
template <typename T, int V>
__device__ __forceinline__ void collide_cells(T (&g)[Q][V], const T omega)
{
#pragma unroll
    for (int j = 0; j < V; ++j) {
        T gc[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) gc[i] = g[i][j];
        collide<T>(gc, omega);
#pragma unroll
        for (int i = 0; i < Q; ++i) g[i][j] = gc[i];
    }
}
// ... or two at a time on the packed fp32 instructions.  Used for fp16
// storage, whose 76 B per update make the kernel issue-bound with scalar
// arithmetic (measured: 11.5 -> 7.1 instructions per cell, 68 -> 70 GLUPS);
// the fp32-storage kernel is memory-bound either way and loses 3 % to the
// extra register pairing, so it keeps the scalar form.
template <int V>
__device__ __forceinline__ void collide_cell_pairs(float (&g)[Q][V], const float omega)
{
    static_assert(V % 2 == 0, "packs hold an even number of cells");
#pragma unroll
    for (int j = 0; j < V; j += 2) {
        float2 gc[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) gc[i] = make_float2(g[i][j], g[i][j + 1]);
        collide<float2>(gc, omega);
#pragma unroll
        for (int i = 0; i < Q; ++i) { g[i][j] = gc[i].x; g[i][j + 1] = gc[i].y; }
    }
}
template <typename TS> struct UsePackedMath { static constexpr bool value = false; };
template <> struct UsePackedMath<__half> { static constexpr bool value = true; };

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

__device__ __forceinline__ void l2_prefetch(const void *p)
{
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// direction table: X(i, c_x, plane offset, row offset)
#define MLB_DIRS(X)                                                              \
    X(1, 1, zc, rc)   X(2, 0, zc, rm)   X(3, -1, zc, rc)  X(4, 0, zc, rq)        \
    X(5, 1, zc, rm)   X(6, -1, zc, rm)  X(7, -1, zc, rq)  X(8, 1, zc, rq)        \
    X(9, 0, zm, rc)   X(10, 0, zq, rc)  X(11, 1, zm, rc)  X(12, -1, zm, rc)      \
    X(13, -1, zq, rc) X(14, 1, zq, rc)  X(15, 0, zm, rm)  X(16, 0, zm, rq)       \
    X(17, 0, zq, rq)  X(18, 0, zq, rm)

// L2 prefetch, one lane per 128-byte line: the lines that the cells `dz` planes
// and `dy` rows further on in launch order (about one wave of resident blocks
// later) will pull (PULL) or find in their own slots (!PULL: the local half of
// the in-place update).  Every value is read exactly once, so this moves no
// extra bytes; it turns that block's DRAM round trip into an L2 hit without
// holding registers for it.  Distances much beyond one wave lose: the
// prefetched lines and the dirty lines of the stores then outgrow L2.
template <typename TS, int V, int LX, bool PULL, typename PTR>
__device__ __forceinline__ void prefetch_ahead(PTR const (&base)[Q], const Geom &gm, int dz,
                                               int dy, int x0, int y, int lz, int lane)
{
    if ((dz | dy) == 0)
        return;
    // (one instruction covers the whole 128-byte line: prefetching per 64 or 32 bytes
    // measures the same)
    constexpr int LPL = 128 / (V * (int)sizeof(TS));   // lanes per line
    int yp = y + dy, lp = lz + dz;
    if (yp >= gm.ny) { yp -= gm.ny; ++lp; }
    if ((lane % LX) % LPL != 0 || lp >= gm.nz)
        return;
    const int xp = (int)gm.xp, plane = (int)gm.plane;
    const int rc = yp * xp, rm = (yp == 0 ? gm.ny - 1 : yp - 1) * xp,
              rq = (yp == gm.ny - 1 ? 0 : yp + 1) * xp;
    const int zc = (lp + 1) * plane + x0;
    const int zm = PULL ? ((lp == 0) ? gm.zlo_src : lp) * plane + x0 : zc;
    const int zq = PULL ? ((lp == gm.nz - 1) ? gm.zhi_src : lp + 2) * plane + x0 : zc;
    l2_prefetch(base[0] + (zc + rc));
#define MLB_X(i, CX, Z, R) l2_prefetch(base[i] + ((Z) + (PULL ? (R) : rc)));
    MLB_DIRS(MLB_X)
#undef MLB_X
}

// The same prefetch as ONE bulk instruction per population and row group
// (cp.async.bulk.prefetch.L2, sm_90+): the rows a block works on are contiguous
// in memory across the whole x extent, so thread i < 19 of the block at
// blockIdx.x == 0 prefetches, for population i, the `nrows` full rows starting at
// row yb (+ the pull's row / plane shift) for all the blocks that share them.
// Rows that wrap around the y edge are left out (they are walls or one row in ny).
constexpr int SEL_zc = 0, SEL_zm = 1, SEL_zq = 2, SEL_rc = 0, SEL_rm = 1, SEL_rq = 2;
template <typename TS, bool PULL, typename PTR>
__device__ __forceinline__ void prefetch_rows(PTR const (&base)[Q], const Geom &gm, int dz, int dy,
                                              int yb, int nrows, int lz, int i)
{
    int r0 = yb + dy, lp = lz + dz;
    if (r0 >= gm.ny) { r0 -= gm.ny; ++lp; }
    if (lp >= gm.nz)
        return;
    int zsel = 0, rsel = 0;
    if (PULL) {
#define MLB_X(ii, CX, Z, R) if (i == ii) { zsel = SEL_##Z; rsel = SEL_##R; }
        MLB_DIRS(MLB_X)
#undef MLB_X
    }
    r0 += rsel == SEL_rm ? -1 : rsel == SEL_rq ? 1 : 0;
    if (r0 < 0) { r0 = 0; --nrows; }
    if (r0 + nrows > gm.ny) nrows = gm.ny - r0;
    if (nrows <= 0)
        return;
    const int zp = zsel == SEL_zc ? lp + 1
                 : zsel == SEL_zm ? (lp == 0 ? gm.zlo_src : lp)
                                  : (lp == gm.nz - 1 ? gm.zhi_src : lp + 2);
    const TS *p = base[i] + ((long long)zp * gm.plane + (long long)r0 * gm.xp);
    const unsigned bytes = (unsigned)(nrows * (int)gm.xp * (int)sizeof(TS));  // whole lines
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(__cvta_generic_to_global(p)),
                 "r"(bytes));
}

// ---------------------------------------------------------------------------
// Fused pull-stream + bounce-back + BGK collide, one thread per cell
// (kernels.py:76-245 `cell`, :247-279 `fused`).  blockIdx = (x tile, y, plane).
// Reads fpre only, writes each FLUID cell of fpost once, nothing else.
//
// The kernel is latency-bound long before it is issue-bound, so everything
// is arranged to put ONE memory round trip on a warp's critical path:
//  * the class word and all 19 pulls are issued together, before the class
//    word is looked at (a solid cell's pulls are simply dropped; wall cells
//    hold valid, never-written populations, so every address is readable);
//  * positions are 32-bit element offsets inside a population
//    (layout_of() guarantees pop < 2^31) on host-computed per-population
//    base pointers: an address is one IMAD + one IMAD.WIDE;
//  * the offset of a source cell is the destination offset plus a
//    BLOCK-UNIFORM delta (y / z neighbours incl. periodic wrap or halo plane)
//    plus a per-thread x delta (-1 / +1, or the wrap distance on edge lanes);
//  * wall-adjacent lanes patch their bounced directions afterwards from the
//    link bits of the class word - no flag reads, no 3-way branches; the
//    patch loads hit lines the same warp has just pulled.
template <typename TS, bool PUSH>
__device__ __forceinline__ void step_cell(const StepArgs<TS> &a, const PushArgs<TS> &ph,
                                          const int x, const int y, const int lz)
{
    using T = typename Store<TS>::C;
    const Geom &gm = a.g;
    const int xp = (int)gm.xp, plane = (int)gm.plane;

    // periodic wrap first, flag test second (kernels.py:83-96)
    const int dxm = (x == 0) ? gm.nx - 1 : -1;            // to the source for c_x = +1
    const int dxq = (x == gm.nx - 1) ? 1 - gm.nx : 1;     // to the source for c_x = -1
    const int rm = ((y == 0) ? gm.ny - 1 : -1) * xp;      // block-uniform row deltas
    const int rq = ((y == gm.ny - 1) ? 1 - gm.ny : 1) * xp;
    const int zm = (((lz == 0) ? gm.zlo_src : lz) - (lz + 1)) * plane;          // plane deltas
    const int zq = (((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) - (lz + 1)) * plane;
    constexpr int zc = 0, rc = 0;

    const int d = (lz + 1) * plane + y * xp + x;
    const int dm = d + dxm, dq = d + dxq, dc = d;

    const uint32_t kd = a.ct.kind[d];
    T g[Q];
    g[0] = Store<TS>::up(a.pre[0][d]);
#define MLB_PULL(i, zz, rr, dd) g[i] = Store<TS>::up(a.pre[i][(dd) + ((zz) + (rr))]);
    MLB_PULL(1, zc, rc, dm)  MLB_PULL(2, zc, rm, dc)  MLB_PULL(3, zc, rc, dq)
    MLB_PULL(4, zc, rq, dc)  MLB_PULL(5, zc, rm, dm)  MLB_PULL(6, zc, rm, dq)
    MLB_PULL(7, zc, rq, dq)  MLB_PULL(8, zc, rq, dm)  MLB_PULL(9, zm, rc, dc)
    MLB_PULL(10, zq, rc, dc) MLB_PULL(11, zm, rc, dm) MLB_PULL(12, zm, rc, dq)
    MLB_PULL(13, zq, rc, dq) MLB_PULL(14, zq, rc, dm) MLB_PULL(15, zm, rm, dc)
    MLB_PULL(16, zm, rq, dc) MLB_PULL(17, zq, rq, dc) MLB_PULL(18, zq, rm, dc)
#undef MLB_PULL
    // one cell per thread: the bulk form, one instruction per population and row
    // (19 per-line prefetches per 32 cells cost too many issue slots here)
    if (blockIdx.x == 0 && threadIdx.x < Q && (a.pf_dz | a.pf_dy) != 0)
        prefetch_rows<TS, true>(a.pre, gm, a.pf_dz, a.pf_dy, y, 1, lz, threadIdx.x);

    // Non-fluid destination.  Strict mode: never written (kernels.py:79-80;
    // the stores of the warp then leave 28-of-32-byte sectors at every wall,
    // which L2 completes with a DRAM read - measured 9 % slower on the
    // cavity).  Pass-through mode: the cell is rewritten with the value it
    // holds in fpre; the caller guarantees fpre and fpost agree on non-fluid
    // cells (true for every state the engine builds: both buffers start
    // identical and only fluid / open-boundary cells ever change), so the
    // bytes in memory are the same as if the cell had not been touched and
    // every store of the warp is a full line.
    const uint32_t cd = kd == 0 ? 0u : cls_of(a.ct, kd, d);
    const bool fluid = (cd & CLS_FLAG) == 0;
    if (!fluid && !a.passthrough)
        return;

    if (fluid) {
        if (cd != 0) {
            // SOLID source -> own opposite population, MOVING_WALL source ->
            // that plus the wall term (kernels.py:88-96)
            const uint32_t mv = (cd & CLS_MOVING) ? mlinks_of(a.ct, kd, d) : 0u;
#pragma unroll
            for (int i = 1; i < Q; ++i)
                if (cd & cls_link(i)) {
                    const T c = Store<TS>::up(a.pre[opp(i)][d]);
                    g[i] = (mv & (1u << i)) ? c + a.k[i] : c;
                }
        }
        collide<T>(g, a.omega);
    } else {
        // pass-through: the pulled values are neighbours', not this cell's
        // (storage -> compute -> storage is exact in every mode)
#pragma unroll
        for (int i = 1; i < Q; ++i)
            g[i] = Store<TS>::up(a.pre[i][d]);
    }

#pragma unroll
    for (int i = 0; i < Q; ++i)
        a.post[i][d] = Store<TS>::down(g[i]);
    if constexpr (PUSH) {
        const int o = y * xp + x;  // offset inside a plane
        if (lz == 0 && ph.lo[0] != nullptr) {
#pragma unroll
            for (int j = 0; j < 5; ++j)
                ph.lo[j][o] = Store<TS>::down(g[halo_down(j)]);
        }
        if (lz == gm.nz - 1 && ph.hi[0] != nullptr) {
#pragma unroll
            for (int j = 0; j < 5; ++j)
                ph.hi[j][o] = Store<TS>::down(g[halo_up(j)]);
        }
    }
}

template <typename TS, int BX, bool PUSH>
__global__ void __launch_bounds__(BX) step_kernel(const StepArgs<TS> a, const PushArgs<TS> ph)
{
    const int x = blockIdx.x * BX + threadIdx.x;
    // pass-through mode also rewrites the row padding: whole last lines (see step_vec_kernel)
    if (x >= (a.passthrough ? (int)a.g.xp : a.g.nx))
        return;
    step_cell<TS, PUSH>(a, ph, x, blockIdx.y, a.z0 + blockIdx.z);
}

// ---------------------------------------------------------------------------
// In-place ("AA pattern") update: ONE population block instead of two, same
// 2 x 19 x sizeof(TS) bytes of traffic per update.  The block alternates
// between two representations of the same post-collision state F:
//   R0 (normal):   A[i][x] = F[i][x]
//   R1 (shifted):  for a fluid cell x and direction i,  F[opp(i)][x] lives at
//                  A[i][x - c_i]   if the cell x - c_i is not a wall,
//                  A[opp(i)][x]    if it is (the link bounces back).
// R0 -> R1 (`aa_pull_kernel`): a cell reads exactly the locations the A/B
// kernel reads (kernels.py:83-197: A[i][x - c_i], or its own A[opp(i)][x]
// (+ wall term) for a bouncing link), collides, and writes the result for
// direction opp(i) back INTO THE LOCATION IT READ for direction i.  Every
// location is read by exactly one cell, so nothing is clobbered.
// R1 -> R0 (`aa_local_kernel`): what a cell needs for direction i is then
// always in its own slot A[opp(i)][x] (the neighbour put it there, or it is
// the cell's own bounced population, which still lacks the wall term - it is
// added here, the same single addition the A/B kernel performs); collide;
// write A[i][x].  Arithmetic and operands are those of the A/B kernel, so
// the populations are bit-identical to it (and to the oracle) after any
// number of steps.  `aa_swap_kernel` converts R1 <-> R0 without a step (for
// diagnostics or a download in the middle of a pair).
// Scope: walls only - flags FLUID / SOLID / MOVING_WALL (open boundaries
// stay on the A/B path), whole domain on one GPU (MLB_Z_PERIODIC).
template <typename TS>
struct AAArgs {
    using T = typename Store<TS>::C;
    TS *f[Q];
    ClsTab ct;
    Geom g;
    T omega;
    T k[Q];
    TS inlet[Q];  // equilibrium(1, u_in, 0, 0), storage dtype (open boundaries, pack kernels)
    int z0;       // first slab plane this launch updates (blockIdx.z = 0)
    int pf_dz, pf_dy;  // L2 prefetch distance of the pack kernels (prefetch_ahead)
    int pf_bulk;
    // z-slabs (REMOTE kernels): the pull half writes each result into the location
    // it was pulled from - and for a boundary plane's crossing directions that
    // location belongs to the ring neighbour.  It is READ from the local halo plane
    // (filled by the previous local half's push, as in the two-buffer path) and
    // WRITTEN straight into the neighbour's boundary plane over peer memory:
    // lo[j] = start of population halo_up(j)'s plane lz = nz_below-1 of the slab
    // below (the source plane of c_z = +1 pulls of our plane 0), hi[j] = start of
    // population halo_down(j)'s plane lz = 0 of the slab above.
    TS *lo[5];
    TS *hi[5];
};
__host__ __device__ constexpr int up_index(int i)    // inverse of halo_up
{ return i == 9 ? 0 : i == 11 ? 1 : i == 12 ? 2 : i == 15 ? 3 : 4; }
__host__ __device__ constexpr int down_index(int i)  // inverse of halo_down
{ return i == 10 ? 0 : i == 13 ? 1 : i == 14 ? 2 : i == 17 ? 3 : 4; }
// c_z of the directions whose source plane is named zc / zm / zq in the tables
constexpr int CZ_zc = 0, CZ_zm = 1, CZ_zq = -1;

// where the pull half stores its result for direction i (source plane offset Z,
// row offset R): the location it read - or the neighbour slab's copy of it
// (x = element offset inside the row; everything is folded into ONE 32-bit offset
// onto a constant-bank base pointer)
template <typename TS, int CZ, bool REMOTE>
__device__ __forceinline__ TS *aa_target(const AAArgs<TS> &a, int i, int Z, int R, int x,
                                         bool rlo, bool rhi)
{
    if (REMOTE && CZ > 0 && rlo) return a.lo[up_index(i)] + (R + x);
    if (REMOTE && CZ < 0 && rhi) return a.hi[down_index(i)] + (R + x);
    return a.f[i] + (Z + R + x);
}

// In place, every non-wall cell takes part in the exchange of slots: fluid cells
// collide; an INLET cell's new state is the constant equilibrium; an OUTLET
// cell's new state is the new state of its x-1 neighbour (engine.py:156-180,
// applied here as part of the step).
__device__ __forceinline__ bool aa_participant(uint32_t c)
{
    const uint32_t fl = c & CLS_FLAG;
    return fl != 1u && fl != 2u;
}

template <typename TS>
struct CellPos {
    int d, off[Q];  // own offset, and the offset of the source cell per direction
};

template <typename TS>
__device__ __forceinline__ void aa_offsets(const Geom &gm, int x, int y, int lz, int &d,
                                           int (&off)[Q])
{
    const int xp = (int)gm.xp, plane = (int)gm.plane;
    const int dxm = (x == 0) ? gm.nx - 1 : -1;
    const int dxq = (x == gm.nx - 1) ? 1 - gm.nx : 1;
    const int rm = ((y == 0) ? gm.ny - 1 : -1) * xp;
    const int rq = ((y == gm.ny - 1) ? 1 - gm.ny : 1) * xp;
    const int zm = (((lz == 0) ? gm.zlo_src : lz) - (lz + 1)) * plane;
    const int zq = (((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) - (lz + 1)) * plane;
    d = (lz + 1) * plane + y * xp + x;
    off[0] = d;
    off[1] = d + dxm;        off[2] = d + rm;         off[3] = d + dxq;        off[4] = d + rq;
    off[5] = d + dxm + rm;   off[6] = d + dxq + rm;   off[7] = d + dxq + rq;   off[8] = d + dxm + rq;
    off[9] = d + zm;         off[10] = d + zq;
    off[11] = d + dxm + zm;  off[12] = d + dxq + zm;  off[13] = d + dxq + zq;  off[14] = d + dxm + zq;
    off[15] = d + rm + zm;   off[16] = d + rq + zm;   off[17] = d + rq + zq;   off[18] = d + rm + zq;
}

// direction table for the scalar in-place kernels: X(i, plane delta, row delta, x-shifted base)
#define MLB_AA_DIRS(X)                                                              \
    X(1, zc, rc, dm)   X(2, zc, rm, dc)   X(3, zc, rc, dq)   X(4, zc, rq, dc)       \
    X(5, zc, rm, dm)   X(6, zc, rm, dq)   X(7, zc, rq, dq)   X(8, zc, rq, dm)       \
    X(9, zm, rc, dc)   X(10, zq, rc, dc)  X(11, zm, rc, dm)  X(12, zm, rc, dq)      \
    X(13, zq, rc, dq)  X(14, zq, rc, dm)  X(15, zm, rm, dc)  X(16, zm, rq, dc)      \
    X(17, zq, rq, dc)  X(18, zq, rm, dc)

template <typename TS, int BX>
__global__ void __launch_bounds__(BX) aa_pull_kernel(const AAArgs<TS> a)
{
    using T = typename Store<TS>::C;
    const Geom &gm = a.g;
    const int x = blockIdx.x * BX + threadIdx.x;
    if (x >= gm.nx)
        return;
    const int y = blockIdx.y, lz = a.z0 + blockIdx.z;
    const int xp = (int)gm.xp, plane = (int)gm.plane;
    // same index arithmetic as step_cell
    const int dxm = (x == 0) ? gm.nx - 1 : -1;
    const int dxq = (x == gm.nx - 1) ? 1 - gm.nx : 1;
    const int rm = ((y == 0) ? gm.ny - 1 : -1) * xp;
    const int rq = ((y == gm.ny - 1) ? 1 - gm.ny : 1) * xp;
    const int zm = (((lz == 0) ? gm.zlo_src : lz) - (lz + 1)) * plane;
    const int zq = (((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) - (lz + 1)) * plane;
    constexpr int zc = 0, rc = 0;
    const int d = (lz + 1) * plane + y * xp + x;
    const int dm = d + dxm, dq = d + dxq, dc = d;

    const uint32_t kd = a.ct.kind[d];
    T g[Q];
    g[0] = Store<TS>::up(a.f[0][d]);
#define MLB_X(i, zz, rr, dd) g[i] = Store<TS>::up(a.f[i][(dd) + ((zz) + (rr))]);
    MLB_AA_DIRS(MLB_X)
#undef MLB_X
    const uint32_t cd = kd == 0 ? 0u : cls_of(a.ct, kd, d);
    if (cd & CLS_FLAG)
        return;
    if (cd != 0) {
        const uint32_t mv = (cd & CLS_MOVING) ? mlinks_of(a.ct, kd, d) : 0u;
#pragma unroll
        for (int i = 1; i < Q; ++i)
            if (cd & cls_link(i)) {
                const T c = Store<TS>::up(a.f[opp(i)][d]);
                g[i] = (mv & (1u << i)) ? c + a.k[i] : c;
            }
    }
    collide<T>(g, a.omega);
    a.f[0][d] = Store<TS>::down(g[0]);
    if (cd == 0) {
        // bulk cell: every result goes into the location read for its opposite
#define MLB_X(i, zz, rr, dd) a.f[i][(dd) + ((zz) + (rr))] = Store<TS>::down(g[opp(i)]);
        MLB_AA_DIRS(MLB_X)
#undef MLB_X
    } else {
#define MLB_X(i, zz, rr, dd)                                                         \
        if (cd & cls_link(i))                                                        \
            a.f[opp(i)][d] = Store<TS>::down(g[opp(i)]); /* bounces: stays, unswapped */ \
        else                                                                         \
            a.f[i][(dd) + ((zz) + (rr))] = Store<TS>::down(g[opp(i)]);
        MLB_AA_DIRS(MLB_X)
#undef MLB_X
    }
}

template <typename TS, int BX>
__global__ void __launch_bounds__(BX) aa_local_kernel(const AAArgs<TS> a)
{
    using T = typename Store<TS>::C;
    const int x = blockIdx.x * BX + threadIdx.x;
    if (x >= a.g.nx)
        return;
    const int d = (a.z0 + (int)blockIdx.z + 1) * (int)a.g.plane + (int)blockIdx.y * (int)a.g.xp + x;
    const uint32_t kd = a.ct.kind[d];
    T g[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i)
        g[i] = Store<TS>::up(a.f[opp(i)][d]);
    const uint32_t cd = kd == 0 ? 0u : cls_of(a.ct, kd, d);
    if (cd & CLS_FLAG) {
        // non-fluid cell: rewrite its own (untouched) values so that every
        // store of the warp is a full line - in place this is always valid
#pragma unroll
        for (int i = 0; i < Q; ++i)
            a.f[opp(i)][d] = Store<TS>::down(g[i]);
        return;
    }
    if (cd & CLS_MOVING) {
        const uint32_t mv = mlinks_of(a.ct, kd, d);
#pragma unroll
        for (int i = 1; i < Q; ++i)
            if (mv & (1u << i))
                g[i] = g[i] + a.k[i];
    }
    collide<T>(g, a.omega);
#pragma unroll
    for (int i = 0; i < Q; ++i)
        a.f[i][d] = Store<TS>::down(g[i]);
}

// R1 <-> R0 without a step: swap each pair of locations {(q, x), (opp(q), x + c_q)}
// whose link does not bounce; each pair is owned by the cell on the "positive"
// side (q in {1,2,5,6,9,11,12,15,16}; x + c_q = the source cell of opp(q)).
template <typename TS, int BX, bool REMOTE>
__global__ void __launch_bounds__(BX) aa_swap_kernel(const AAArgs<TS> a)
{
    const int x = blockIdx.x * BX + threadIdx.x;
    if (x >= a.g.nx)
        return;
    const int lz = a.z0 + blockIdx.z;
    int d, off[Q];
    aa_offsets<TS>(a.g, x, blockIdx.y, lz, d, off);
    const uint32_t kd = a.ct.kind[d];
    const uint32_t cd = kd == 0 ? 0u : cls_of(a.ct, kd, d);
    if (!aa_participant(cd))
        return;
    // z-slabs: the partner of a top-plane cell along a c_z = +1 direction lives in
    // the slab above (its plane 0), not in our halo
    const bool rhi = REMOTE && lz == a.g.nz - 1 && a.hi[0] != nullptr;
    const int halo_hi = a.g.zhi_src * (int)a.g.plane;
#pragma unroll
    for (int q = 1; q < Q; ++q) {
        const bool positive = (q == 1 || q == 2 || q == 5 || q == 6 || q == 9 || q == 11
                               || q == 12 || q == 15 || q == 16);
        if (!positive)
            continue;
        const int o = opp(q);           // x + c_q is the source cell of direction o
        if (cd & cls_link(o))
            continue;                   // bouncing link: both representations agree
        const bool up = (q == 9 || q == 11 || q == 12 || q == 15 || q == 16);  // c_z(q) = +1
        TS *partner = (up && rhi) ? a.hi[down_index(o)] + (off[o] - halo_hi) : a.f[o] + off[o];
        const TS u = a.f[q][d], v = *partner;
        a.f[q][d] = v;
        *partner = u;
    }
}

// ---------------------------------------------------------------------------
// Vectorised variant: each thread owns a PACK of V consecutive cells in x
// (one 16-byte word per population in fp32 / fp64, 8 or 4 bytes in fp16
// storage); a warp covers LX
// packs in x by 32 / LX rows in y.  Per pack and population: one aligned
// 16-byte load; the ten populations with c_x = +-1 need the word shifted by
// one cell, which costs one extra scalar load of the element just outside
// the pack (an L1 hit: the neighbouring lane's word holds it).  Stores are
// aligned 16-byte words (pull scheme: destinations are never shifted).
// Same early-issue and link-bit patching as the scalar kernel.  Kept as a
// selectable variant: at 512^3 it measures within 2 % of the scalar kernel
// (fewer instructions per cell, but 3x the registers per thread).
// pack loads / stores: V consecutive storage elements <-> V compute values
template <typename TS, int V> struct PackIO;
template <> struct PackIO<float, 4> {
    static __device__ __forceinline__ void load(const float *p, float (&o)[4])
    { const float4 v = *reinterpret_cast<const float4 *>(p); o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w; }
    static __device__ __forceinline__ void store(float *p, const float (&o)[4])
    { *reinterpret_cast<float4 *>(p) = make_float4(o[0], o[1], o[2], o[3]); }
    // all but the last / all but the first cell of the pack, in the widest aligned pieces
    // (the in-place pull half at the ends of a warp row; `full` picks the whole pack instead)
    static __device__ __forceinline__ void store_head(float *p, const float (&o)[4], bool full)
    {
        if (full) { store(p, o); return; }
        *reinterpret_cast<float2 *>(p) = make_float2(o[0], o[1]);
        p[2] = o[2];
    }
    static __device__ __forceinline__ void store_tail(float *p, const float (&o)[4], bool full)
    {
        if (full) { store(p, o); return; }
        p[1] = o[1];
        *reinterpret_cast<float2 *>(p + 2) = make_float2(o[2], o[3]);
    }
};
template <> struct PackIO<float, 2> {   // 8-byte packs: rows whose length is even but not a multiple of 4
    static __device__ __forceinline__ void load(const float *p, float (&o)[2])
    { const float2 v = *reinterpret_cast<const float2 *>(p); o[0] = v.x; o[1] = v.y; }
    static __device__ __forceinline__ void store(float *p, const float (&o)[2])
    { *reinterpret_cast<float2 *>(p) = make_float2(o[0], o[1]); }
    static __device__ __forceinline__ void store_head(float *p, const float (&o)[2], bool full)
    { if (full) store(p, o); else p[0] = o[0]; }
    static __device__ __forceinline__ void store_tail(float *p, const float (&o)[2], bool full)
    { if (full) store(p, o); else p[1] = o[1]; }
};
template <> struct PackIO<double, 2> {
    static __device__ __forceinline__ void load(const double *p, double (&o)[2])
    { const double2 v = *reinterpret_cast<const double2 *>(p); o[0] = v.x; o[1] = v.y; }
    static __device__ __forceinline__ void store(double *p, const double (&o)[2])
    { *reinterpret_cast<double2 *>(p) = make_double2(o[0], o[1]); }
    static __device__ __forceinline__ void store_head(double *p, const double (&o)[2], bool full)
    { if (full) store(p, o); else p[0] = o[0]; }
    static __device__ __forceinline__ void store_tail(double *p, const double (&o)[2], bool full)
    { if (full) store(p, o); else p[1] = o[1]; }
};
template <> struct PackIO<f32w, 2> {
    static __device__ __forceinline__ void load(const f32w *p, double (&o)[2])
    { const float2 v = *reinterpret_cast<const float2 *>(p); o[0] = (double)v.x; o[1] = (double)v.y; }
    static __device__ __forceinline__ void store(f32w *p, const double (&o)[2])
    { *reinterpret_cast<float2 *>(p) = make_float2((float)o[0], (float)o[1]); }
    static __device__ __forceinline__ void store_head(f32w *p, const double (&o)[2], bool full)
    {
        const float2 r = make_float2((float)o[0], (float)o[1]);   // one rounding per value either way
        if (full) *reinterpret_cast<float2 *>(p) = r; else p[0].v = r.x;
    }
    static __device__ __forceinline__ void store_tail(f32w *p, const double (&o)[2], bool full)
    {
        const float2 r = make_float2((float)o[0], (float)o[1]);
        if (full) *reinterpret_cast<float2 *>(p) = r; else p[1].v = r.y;
    }
};
template <> struct PackIO<__half, 2> {
    static __device__ __forceinline__ void load(const __half *p, float (&o)[2])
    { const __half2 v = *reinterpret_cast<const __half2 *>(p); o[0] = __low2float(v); o[1] = __high2float(v); }
    static __device__ __forceinline__ void store(__half *p, const float (&o)[2])
    { *reinterpret_cast<__half2 *>(p) = __floats2half2_rn(o[0], o[1]); }
    static __device__ __forceinline__ void store_head(__half *p, const float (&o)[2], bool full)
    {
        const __half2 r = __floats2half2_rn(o[0], o[1]);
        if (full) *reinterpret_cast<__half2 *>(p) = r; else p[0] = __low2half(r);
    }
    static __device__ __forceinline__ void store_tail(__half *p, const float (&o)[2], bool full)
    {
        const __half2 r = __floats2half2_rn(o[0], o[1]);
        if (full) *reinterpret_cast<__half2 *>(p) = r; else p[1] = __high2half(r);
    }
};
template <> struct PackIO<__half, 4> {
    static __device__ __forceinline__ void load(const __half *p, float (&o)[4])
    {
        const uint2 u = *reinterpret_cast<const uint2 *>(p);
        const __half2 a = *reinterpret_cast<const __half2 *>(&u.x);
        const __half2 b = *reinterpret_cast<const __half2 *>(&u.y);
        o[0] = __low2float(a); o[1] = __high2float(a); o[2] = __low2float(b); o[3] = __high2float(b);
    }
    static __device__ __forceinline__ void store(__half *p, const float (&o)[4])
    {
        const __half2 a = __floats2half2_rn(o[0], o[1]), b = __floats2half2_rn(o[2], o[3]);
        uint2 u;
        u.x = *reinterpret_cast<const unsigned *>(&a);
        u.y = *reinterpret_cast<const unsigned *>(&b);
        *reinterpret_cast<uint2 *>(p) = u;
    }
    // the two packed words are converted ONCE (F2FP) whichever pieces get stored
    static __device__ __forceinline__ void store_head(__half *p, const float (&o)[4], bool full)
    {
        const __half2 a = __floats2half2_rn(o[0], o[1]), b = __floats2half2_rn(o[2], o[3]);
        if (full) {
            uint2 u;
            u.x = *reinterpret_cast<const unsigned *>(&a);
            u.y = *reinterpret_cast<const unsigned *>(&b);
            *reinterpret_cast<uint2 *>(p) = u;
        } else {
            *reinterpret_cast<__half2 *>(p) = a;
            p[2] = __low2half(b);
        }
    }
    static __device__ __forceinline__ void store_tail(__half *p, const float (&o)[4], bool full)
    {
        const __half2 a = __floats2half2_rn(o[0], o[1]), b = __floats2half2_rn(o[2], o[3]);
        if (full) {
            uint2 u;
            u.x = *reinterpret_cast<const unsigned *>(&a);
            u.y = *reinterpret_cast<const unsigned *>(&b);
            *reinterpret_cast<uint2 *>(p) = u;
        } else {
            p[1] = __high2half(a);
            *reinterpret_cast<__half2 *>(p + 2) = b;
        }
    }
};
// the kind bytes of a pack, as one word (byte j = cell j)
template <int V> struct KindIO;
template <> struct KindIO<2> {
    static __device__ __forceinline__ uint32_t load(const uint8_t *p)
    { return *reinterpret_cast<const uint16_t *>(p); }
};
template <> struct KindIO<4> {
    static __device__ __forceinline__ uint32_t load(const uint8_t *p)
    { return *reinterpret_cast<const uint32_t *>(p); }
};

// The V values pulled along a direction with x component CX from the row
// starting at `row` (already offset to population, plane and row).
template <typename TS, int V, int CX>
__device__ __forceinline__ void pull_pack(const TS *__restrict__ row, int x0, int xl, int xr,
                                          typename Store<TS>::C (&o)[V])
{
    typename Store<TS>::C w[V];
    PackIO<TS, V>::load(row + x0, w);
    if (CX == 0) {
#pragma unroll
        for (int j = 0; j < V; ++j) o[j] = w[j];
    } else if (CX > 0) {  // source x - 1
        o[0] = Store<TS>::up(row[xl]);
#pragma unroll
        for (int j = 1; j < V; ++j) o[j] = w[j - 1];
    } else {              // source x + 1
#pragma unroll
        for (int j = 0; j < V - 1; ++j) o[j] = w[j + 1];
        o[V - 1] = Store<TS>::up(row[xr]);
    }
}

// What follows the loads of a pack, shared by the direct kernel (step_vec_kernel)
// and the staged one (step_stage_kernel): class words, link-bit patching, collide,
// pass-through / open-boundary substitution, stores, fused halo push.  `g` holds
// the pulled populations of the pack's V cells, `kpack` their kind bytes, `d` the
// pack's offset inside a population, `o_plane` its offset inside the plane.
template <typename TS, int V, bool PUSH>
__device__ __forceinline__ void vec_finish(const StepArgs<TS> &a, const PushArgs<TS> &ph,
                                           typename Store<TS>::C (&g)[Q][V], const uint32_t kpack,
                                           const int d, const int o_plane, const int lz)
{
    using T = typename Store<TS>::C;
    const Geom &gm = a.g;
    // class words: all zero for a pack of bulk cells (the usual case), else from
    // the dictionary.  (A separate code path for bulk packs was measured and is
    // slower: warps that mix bulk and wall packs then run the collide twice.)
    uint32_t c[V];
#pragma unroll
    for (int j = 0; j < V; ++j)
        c[j] = 0u;
    if (kpack != 0u) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint32_t k = (kpack >> (8 * j)) & 0xffu;
            if (k != 0u)
                c[j] = cls_of(a.ct, k, d + j);
        }
    }
    uint32_t call = 0u;
    bool anyfluid = false, allfluid = true;
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const bool fl = (c[j] & CLS_FLAG) == 0;
        anyfluid |= fl;
        allfluid &= fl;
        call |= fl ? c[j] : 0u;
    }
    if (!anyfluid && !a.passthrough)
        return;

    if (call != 0) {  // some fluid cell of the pack touches a wall
        uint32_t mv[V];
#pragma unroll
        for (int j = 0; j < V; ++j)
            mv[j] = ((c[j] & CLS_FLAG) == 0 && (c[j] & CLS_MOVING))
                        ? mlinks_of(a.ct, (kpack >> (8 * j)) & 0xffu, d + j) : 0u;
#pragma unroll
        for (int i = 1; i < Q; ++i)
            if (call & cls_link(i)) {
                T o[V];
                PackIO<TS, V>::load(a.pre[opp(i)] + d, o);
#pragma unroll
                for (int j = 0; j < V; ++j)
                    if (c[j] & cls_link(i))
                        g[i][j] = (mv[j] & (1u << i)) ? o[j] + a.k[i] : o[j];
            }
    }

    // collide the cells of the pack (lattice.collide_cell order; two cells per
    // packed-fp32 instruction when computing in float)
    if constexpr (UsePackedMath<TS>::value)
        collide_cell_pairs<V>(g, a.omega);
    else
        collide_cells<T, V>(g, a.omega);

    if (!allfluid && a.passthrough) {
        // non-fluid cells of the pack keep the value they hold in fpre
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            T o[V];
            PackIO<TS, V>::load(a.pre[i] + d, o);
#pragma unroll
            for (int j = 0; j < V; ++j)
                if ((c[j] & CLS_FLAG) != 0)
                    g[i][j] = o[j];
        }
        if (a.fuse_open) {
            // _OpenBoundaryPass.apply fused into the store: inlet cells take the
            // constant equilibrium; then outlet cells take the fresh value of
            // their x-1 neighbour - a cell of the same pack (the host checked
            // that no outlet cell starts a pack).  Descending j reads each left
            // neighbour before it could itself be substituted, which is numpy's
            // "right-hand side first" (engine.py:179-180).
#pragma unroll
            for (int j = 0; j < V; ++j)
                if ((c[j] & CLS_FLAG) == 3) {
#pragma unroll
                    for (int i = 0; i < Q; ++i)
                        g[i][j] = Store<TS>::up(a.inlet[i]);
                }
#pragma unroll
            for (int j = V - 1; j >= 1; --j)
                if ((c[j] & CLS_FLAG) == 4) {
#pragma unroll
                    for (int i = 0; i < Q; ++i)
                        g[i][j] = g[i][j - 1];
                }
        }
    }
    if (allfluid || a.passthrough) {
#pragma unroll
        for (int i = 0; i < Q; ++i)
            PackIO<TS, V>::store(a.post[i] + d, g[i]);
    } else {
#pragma unroll
        for (int j = 0; j < V; ++j)
            if ((c[j] & CLS_FLAG) == 0) {
#pragma unroll
                for (int i = 0; i < Q; ++i)
                    a.post[i][d + j] = Store<TS>::down(g[i][j]);
            }
    }
    if constexpr (PUSH) {
        // the crossing populations of a boundary plane, also into the ring
        // neighbour's halo plane (peer memory): same values, same cells
        const bool lo = lz == 0 && ph.lo[0] != nullptr;
        const bool hi = lz == gm.nz - 1 && ph.hi[0] != nullptr;
        if (lo || hi) {
            const int o = o_plane;
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                if (allfluid || a.passthrough) {
                    if (lo) PackIO<TS, V>::store(ph.lo[j] + o, g[halo_down(j)]);
                    if (hi) PackIO<TS, V>::store(ph.hi[j] + o, g[halo_up(j)]);
                } else {
#pragma unroll
                    for (int jj = 0; jj < V; ++jj)
                        if ((c[jj] & CLS_FLAG) == 0) {
                            if (lo) ph.lo[j][o + jj] = Store<TS>::down(g[halo_down(j)][jj]);
                            if (hi) ph.hi[j][o + jj] = Store<TS>::down(g[halo_up(j)][jj]);
                        }
                }
            }
        }
    }
}

template <typename TS, int V, int LX, bool PUSH>
__global__ void __launch_bounds__(128, 4) step_vec_kernel(const StepArgs<TS> a,
                                                          const PushArgs<TS> ph)
{
    using T = typename Store<TS>::C;
    constexpr int RPW = 32 / LX;        // rows per warp
    const Geom &gm = a.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * LX + (lane % LX)) * V;
    const int y = blockIdx.y * (4 * RPW) + warp * RPW + lane / LX;
    const int lz = a.z0 + blockIdx.z;
    const int xp = (int)gm.xp, plane = (int)gm.plane;
    // Pass-through mode also rewrites the row padding (kind 1: "solid", holds
    // whatever the block was allocated with, read by nobody): the last line of a
    // row whose length is not a multiple of 128 bytes is then stored whole instead
    // of leaving a partial sector for L2 to complete with a DRAM read.
    if (x0 >= (a.passthrough ? xp : gm.nx) || y >= gm.ny)
        return;

    const int zc = (lz + 1) * plane;
    const int zm = ((lz == 0) ? gm.zlo_src : lz) * plane;
    const int zq = ((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) * plane;
    const int ym = (y == 0) ? gm.ny - 1 : y - 1;
    const int yq = (y == gm.ny - 1) ? 0 : y + 1;
    const int rc = y * xp, rm = ym * xp, rq = yq * xp;
    const int xl = (x0 == 0) ? gm.nx - 1 : x0 - 1;
    const int xr = (x0 + V >= gm.nx) ? 0 : x0 + V;
    const int d = zc + rc + x0;

    // kind bytes of the pack and all pulls, issued together
    const uint32_t kpack = KindIO<V>::load(a.ct.kind + d);
    T g[Q][V];
    PackIO<TS, V>::load(a.pre[0] + d, g[0]);
#define MLB_X(i, CX, Z, R) pull_pack<TS, V, CX>(a.pre[i] + ((Z) + (R)), x0, xl, xr, g[i]);
    MLB_DIRS(MLB_X)
#undef MLB_X
    // rows whose length the pack does not divide: the cell at x = nx-1 sits inside
    // the last pack, and its x+1 neighbour is cell 0 of the row, not the padding
    if (x0 + V > gm.nx) {
        const int js = gm.nx - 1 - x0;
#define MLB_X(i, CX, Z, R)                                                           \
        if (CX < 0) {                                                                \
            const T w0 = Store<TS>::up((a.pre[i] + ((Z) + (R)))[0]);                 \
            _Pragma("unroll") for (int j = 0; j < V - 1; ++j)                        \
                if (j == js) g[i][j] = w0;                                           \
        }
        MLB_DIRS(MLB_X)
#undef MLB_X
    }

    if (a.pf_bulk) {
        if (blockIdx.x == 0 && threadIdx.x < Q && (a.pf_dz | a.pf_dy) != 0)
            prefetch_rows<TS, true>(a.pre, gm, a.pf_dz, a.pf_dy, blockIdx.y * (4 * RPW), 4 * RPW, lz,
                                    threadIdx.x);
    } else
        prefetch_ahead<TS, V, LX, true>(a.pre, gm, a.pf_dz, a.pf_dy, x0, y, lz, lane);

    vec_finish<TS, V, PUSH>(a, ph, g, kpack, d, rc + x0, lz);
}

// ---------------------------------------------------------------------------
// Staged variant (the north star's "shared-memory ... staging of the neighbour
// planes"): every WARP is its own software pipeline.  A warp owns a column of
// 32 packs (32 V cells) and walks `rows` consecutive rows of one plane; the 19
// row segments the next row's cells pull from (shifted by the direction's y / z
// component - periodic wrap or halo plane exactly as in the direct kernel - plus
// one 16-byte chunk either side for the x shift, the periodic wrap in x
// included) and the kind bytes travel global -> shared memory with cp.async
// (LDGSTS: no register is held while the bytes are in flight), two rows ahead
// of the arithmetic:
//     issue row t+1   ->   wait for row t   ->   shared -> registers   ->
//     patch / collide / store (vec_finish: the direct kernel's code, same bits)
// No block-level barrier, only __syncwarp: warps drift freely, as in the direct
// kernel.  What it buys over the direct kernel: the loads of the next row are in
// flight during the whole arithmetic phase instead of an L2 prefetch that only
// shortens the round trip; what it costs: 29 shared-memory loads per pack.
// (A first version staged whole-row tiles per BLOCK with cp.async.bulk + mbarrier:
// bit-exact too, but the block-wide phases left the SM idle two thirds of the
// time - 41 instead of 72 GLUPS with fp16 storage at 512^3.)
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc, bool pred)
{
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %2, 0;\n"
#ifdef MLB_STAGE_CA
        "@p cp.async.ca.shared.global [%0], [%1], 16;\n"
#else
        "@p cp.async.cg.shared.global [%0], [%1], 16;\n"
#endif
        "}\n" ::"r"(d), "l"(gsrc), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename TS, int V>
struct StageShape {
    static constexpr int E = 16 / (int)sizeof(TS);          // elements per 16-byte chunk
    static constexpr int W = 32 * V;                         // cells per warp row
    static constexpr int SLICE = W + 2 * E;                  // elements per staged segment
    static constexpr int CHUNKS = SLICE / E;                 // 16-byte chunks per segment (<= 32)
    static constexpr int KCHUNKS = W / 16;                   // chunks of kind bytes
    static constexpr int STAGE_BYTES = Q * SLICE * (int)sizeof(TS) + W;
    static constexpr int WARP_BYTES = 2 * STAGE_BYTES;       // two rows in flight / in use
    // one lane per chunk: the modes this kernel is meant for (fp16 storage, fp32
    // storage with fp64 arithmetic: 256-byte warp rows); fp32 / fp64 run at the HBM
    // roofline with the direct kernel
    static constexpr bool OK = CHUNKS <= 32;
    static_assert(STAGE_BYTES % 16 == 0, "stages stay 16-byte aligned");
};

template <typename TS, int V>
__global__ void __launch_bounds__(128, 4)
step_stage_kernel(const StepArgs<TS> a, const int group, const int ncol, const int ntasks)
{
    using T = typename Store<TS>::C;
    using SS = StageShape<TS, V>;
    static_assert(SS::OK, "a staged segment must fit one cp.async per lane");
    extern __shared__ __align__(128) unsigned char stage_mem[];
    const Geom &gm = a.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int xp = (int)gm.xp, plane = (int)gm.plane;
    unsigned char *mine = stage_mem + (size_t)warp * SS::WARP_BYTES;
    constexpr bool KSAME = SS::CHUNKS + SS::KCHUNKS <= 32;
    const int klane = KSAME ? lane - SS::CHUNKS : lane;
    const PushArgs<TS> noph{};

    // Work units are warp rows - (column of 32 packs, row, plane), column fastest - handed
    // out IN ORDER, `group` at a time, from one counter: whichever warp is free takes the
    // next ones, so the warps in flight always work on one compact window of the domain
    // that sweeps through memory in address order, exactly like the blocks of the direct
    // kernel under the hardware scheduler.  (A static assignment - every warp walking its
    // own 16 rows - was measured at HALF the speed: the windows drift apart and DRAM page
    // locality goes; the same happened to every looped kernel tried in round 1 and 2.)
    int ubase = 0, uk = group;
    auto next_unit = [&]() -> int {
        if (uk == group) {
            unsigned int gidx = 0;
            if (lane == 0) gidx = atomicAdd(a.work, 1u);
            gidx = __shfl_sync(0xffffffffu, gidx, 0);
            ubase = gidx > 0x3fffffffu / (unsigned)group ? ntasks : (int)gidx * group;
            uk = 0;
        }
        const int u = ubase + uk++;
        return u < ntasks ? u : ntasks;
    };
    struct Unit { int xw, y, lz; };
    auto locate = [&](int u) -> Unit {
        const int col = u % ncol, rest = u / ncol;
        return Unit{col * SS::W, rest % gm.ny, a.z0 + rest / gm.ny};
    };

    auto fetch = [&](const Unit &w, int st) {
        TS *seg = reinterpret_cast<TS *>(mine + (size_t)st * SS::STAGE_BYTES);
        const int lz = w.lz, y = w.y, xw = w.xw;
        const int zc = (lz + 1) * plane;
        const int zm = ((lz == 0) ? gm.zlo_src : lz) * plane;
        const int zq = ((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) * plane;
        const int ym = (y == 0) ? gm.ny - 1 : y - 1;
        const int yq = (y == gm.ny - 1) ? 0 : y + 1;
        const int rc = y * xp, rm = ym * xp, rq = yq * xp;
        // chunk `lane` of a segment: elements [xw - E + lane E, + E) of the source row,
        // the outer two wrapped around the row (periodic in x) where the column touches
        // its ends; chunks past the padded row are not fetched (nobody reads them)
        int coff = xw - SS::E + lane * SS::E;
        if (lane == 0 && xw == 0) coff = ((gm.nx - 1) / SS::E) * SS::E;
        if (lane == SS::CHUNKS - 1 && xw + SS::W >= gm.nx) coff = 0;
        const bool cpred = lane < SS::CHUNKS && coff >= 0 && coff < xp;
        const bool kpred = klane >= 0 && klane < SS::KCHUNKS && xw + klane * 16 < xp;
        cp_async16(seg + lane * SS::E, a.pre[0] + (zc + rc + coff), cpred);
#define MLB_X(i, CX, Z, R)                                                           \
        cp_async16(seg + i * SS::SLICE + lane * SS::E, a.pre[i] + ((Z) + (R) + coff), cpred);
        MLB_DIRS(MLB_X)
#undef MLB_X
        unsigned char *kd = reinterpret_cast<unsigned char *>(seg + Q * SS::SLICE);
        cp_async16(kd + klane * 16, a.ct.kind + (zc + rc + xw + klane * 16), kpred);
        cp_async_commit();
        // (optional) the L2 prefetch of the direct kernel on top: the staged copies
        // then find their lines in L2
        prefetch_ahead<TS, V, 32, true>(a.pre, gm, a.pf_dz, a.pf_dy, xw + lane * V, y, lz, lane);
    };

    int u_cur = next_unit();
    if (u_cur >= ntasks)
        return;
    Unit cur = locate(u_cur);
    fetch(cur, 0);
    for (int st = 0;; st ^= 1) {
        const int u_nxt = next_unit();
        Unit nxt{0, 0, 0};
        if (u_nxt < ntasks) {
            nxt = locate(u_nxt);
            fetch(nxt, st ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncwarp();
        const int x0 = cur.xw + lane * V;
        const bool active = x0 < (a.passthrough ? xp : gm.nx);
        // positions inside a staged segment: own pack, the cell left of it, the cell right of it
        const int p = SS::E + lane * V;
        const int pl = (x0 == 0) ? (gm.nx - 1) % SS::E : p - 1;
        const int pr = (x0 + V >= gm.nx) ? SS::E + SS::W : p + V;
        const TS *seg = reinterpret_cast<const TS *>(mine + (size_t)st * SS::STAGE_BYTES);
        uint32_t kpack = 0u;
        T g[Q][V];
        if (active) {
            kpack = KindIO<V>::load(reinterpret_cast<const uint8_t *>(seg + Q * SS::SLICE) + lane * V);
            PackIO<TS, V>::load(seg + p, g[0]);
#define MLB_X(i, CX, Z, R) pull_pack<TS, V, CX>(seg + i * SS::SLICE, p, pl, pr, g[i]);
            MLB_DIRS(MLB_X)
#undef MLB_X
            if (x0 + V > gm.nx) {   // the pack that holds x = nx-1 of a ragged row (see step_vec_kernel)
                const int js = gm.nx - 1 - x0;
#define MLB_X(i, CX, Z, R)                                                           \
                if (CX < 0) {                                                        \
                    const T w0 = Store<TS>::up((seg + i * SS::SLICE)[SS::E + SS::W]); \
                    _Pragma("unroll") for (int j = 0; j < V - 1; ++j)                \
                        if (j == js) g[i][j] = w0;                                   \
                }
                MLB_DIRS(MLB_X)
#undef MLB_X
            }
        }
        __syncwarp();               // every lane holds its pack: the stage may be refilled
        if (active) {
            const int o_plane = cur.y * xp + x0;
            vec_finish<TS, V, false>(a, noph, g, kpack, (cur.lz + 1) * plane + o_plane, o_plane,
                                     cur.lz);
        }
        if (u_nxt >= ntasks)
            break;
        cur = nxt;
    }
}

// ---------------------------------------------------------------------------
// Vectorised in-place kernels: the thread / warp layout, loads, link-bit
// patching and collide of step_vec_kernel; what differs is where results go.
//
// aa_pull_vec_kernel (R0 -> R1).  A cell writes its result for opp(i) into
// the location it read for i: A[i][x - c_i] (or its own A[opp(i)][x] when the
// link bounces).  For the 8 directions with c_x = 0 that is an aligned pack
// in a neighbouring row / plane.  For the 10 directions with c_x = +-1 the
// pack is shifted by one cell; to keep every store an aligned 16-byte word, a
// lane stores the aligned pack made of its own cells' results (all but one)
// plus ONE value from the neighbouring lane (a warp shuffle): with c_x = +1
// lane L stores the results of cells x0+1 .. x0+V (its cells 1..V-1 and the
// right lane's cell 0) at A[i][x0 .. x0+V-1].  That is only valid when every
// cell involved is a bulk fluid cell (kind 0: no bouncing link, so each of
// these locations has exactly this one writer); both lanes know both kind
// words (a shuffled predicate), so they agree on who writes what: if either
// pack is not all-bulk, or the neighbour is in another warp row, each lane
// falls back to per-cell stores for its own cells, with the scalar kernel's
// rules.  Every location still has exactly one writer.
// resident blocks per SM the register allocation aims at (measured: fp64 is
// better off with 168 registers and no spills, fp32 / fp16 storage with 128)
template <typename TS> struct AaMinBlocks { static constexpr int value = 4; };
template <> struct AaMinBlocks<double> { static constexpr int value = 3; };
// WPR > 0 selects the ROW-BLOCK layout: a warp is one row segment of 32 packs, the
// block's four warps are WPR segments side by side in x times 4 / WPR rows, and
// the one value (and the bulk flag) that crosses a WARP boundary travels through
// shared memory - so a block that spans the whole row (nx = WPR * 32 * V, the
// periodic wrap included) has no row ends at all, and every store of a bulk pack
// is an aligned pack; a longer row has ends only at block boundaries.
template <typename TS, int V, int LX, bool REMOTE, int WPR = 0>
__global__ void __launch_bounds__(128, AaMinBlocks<TS>::value)
aa_pull_vec_kernel(const AAArgs<TS> a)
{
    using T = typename Store<TS>::C;
    constexpr bool ROWB = WPR > 0;
    constexpr int LXE = ROWB ? 32 : LX;          // packs per warp row
    constexpr int RPW = 32 / LXE;
    constexpr int BROWS = ROWB ? 4 / (WPR > 0 ? WPR : 1) : 4 * RPW;   // rows per block
    constexpr unsigned FULL = 0xffffffffu;
    const Geom &gm = a.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int seg = lane % LXE;
    const int wseg = ROWB ? warp % (WPR > 0 ? WPR : 1) : 0;   // the warp's segment of the block row
    int x0 = ROWB ? ((blockIdx.x * WPR + wseg) * 32 + lane) * V : (blockIdx.x * LX + seg) * V;
    int y = ROWB ? blockIdx.y * BROWS + warp / (WPR > 0 ? WPR : 1)
                 : blockIdx.y * (4 * RPW) + warp * RPW + lane / LXE;
    const int lz = a.z0 + blockIdx.z;
    // z-slabs: crossing directions of a boundary plane store into the neighbour slab
    const bool rlo = REMOTE && lz == 0 && a.lo[0] != nullptr;
    const bool rhi = REMOTE && lz == gm.nz - 1 && a.hi[0] != nullptr;
    // lanes outside the grid stay in the warp for the shuffles: they compute on
    // a valid dummy pack and never store
    const bool valid = x0 < gm.nx && y < gm.ny;
    if (!valid) { x0 = 0; y = 0; }

    const int xp = (int)gm.xp, plane = (int)gm.plane;
    const int zc = (lz + 1) * plane;
    const int zm = ((lz == 0) ? gm.zlo_src : lz) * plane;
    const int zq = ((lz == gm.nz - 1) ? gm.zhi_src : lz + 2) * plane;
    const int ym = (y == 0) ? gm.ny - 1 : y - 1;
    const int yq = (y == gm.ny - 1) ? 0 : y + 1;
    const int rc = y * xp, rm = ym * xp, rq = yq * xp;
    const int xl = (x0 == 0) ? gm.nx - 1 : x0 - 1;
    const int xr = (x0 + V >= gm.nx) ? 0 : x0 + V;
    const int d = zc + rc + x0;

    const uint32_t kpack = KindIO<V>::load(a.ct.kind + d);
    T g[Q][V];
    PackIO<TS, V>::load(a.f[0] + d, g[0]);
#define MLB_X(i, CX, Z, R) pull_pack<TS, V, CX>(a.f[i] + ((Z) + (R)), x0, xl, xr, g[i]);
    MLB_DIRS(MLB_X)
#undef MLB_X
    if (x0 + V > gm.nx) {   // the pack that holds x = nx-1 of a ragged row (see step_vec_kernel)
        const int js = gm.nx - 1 - x0;
#define MLB_X(i, CX, Z, R)                                                           \
        if (CX < 0) {                                                                \
            const T w0 = Store<TS>::up((a.f[i] + ((Z) + (R)))[0]);                   \
            _Pragma("unroll") for (int j = 0; j < V - 1; ++j)                        \
                if (j == js) g[i][j] = w0;                                           \
        }
        MLB_DIRS(MLB_X)
#undef MLB_X
    }
    if (a.pf_bulk) {
        if (blockIdx.x == 0 && threadIdx.x < Q && (a.pf_dz | a.pf_dy) != 0)
            prefetch_rows<TS, true>(a.f, gm, a.pf_dz, a.pf_dy, blockIdx.y * BROWS, BROWS, lz,
                                    threadIdx.x);
    } else
        prefetch_ahead<TS, V, LXE, true>(a.f, gm, a.pf_dz, a.pf_dy, x0, y, lz, lane);

    const bool bulk = valid && kpack == 0u;
    bool bulk_r = __shfl_down_sync(FULL, (int)bulk, 1) != 0 && seg != LXE - 1
                  && x0 + V < gm.nx;
    bool bulk_l = __shfl_up_sync(FULL, (int)bulk, 1) != 0 && seg != 0;

    uint32_t c[V];
#pragma unroll
    for (int j = 0; j < V; ++j)
        c[j] = 0u;
    if (kpack != 0u) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint32_t k = (kpack >> (8 * j)) & 0xffu;
            if (k != 0u)
                c[j] = cls_of(a.ct, k, d + j);
        }
    }
    uint32_t call = 0u;
#pragma unroll
    for (int j = 0; j < V; ++j)
        call |= ((c[j] & CLS_FLAG) == 0) ? c[j] : 0u;
    if (call != 0) {
        uint32_t mv[V];
#pragma unroll
        for (int j = 0; j < V; ++j)
            mv[j] = ((c[j] & CLS_FLAG) == 0 && (c[j] & CLS_MOVING))
                        ? mlinks_of(a.ct, (kpack >> (8 * j)) & 0xffu, d + j) : 0u;
#pragma unroll
        for (int i = 1; i < Q; ++i)
            if (call & cls_link(i)) {
                T o[V];
                PackIO<TS, V>::load(a.f[opp(i)] + d, o);
#pragma unroll
                for (int j = 0; j < V; ++j)
                    if (c[j] & cls_link(i))
                        g[i][j] = (mv[j] & (1u << i)) ? o[j] + a.k[i] : o[j];
            }
    }
    if constexpr (UsePackedMath<TS>::value)
        collide_cell_pairs<V>(g, a.omega);
    else
        collide_cells<T, V>(g, a.omega);

    // open-boundary cells of the pack: their new state by rule instead of by
    // collision (same order as the fused two-buffer pass: walls hold their own
    // values, inlet cells the constant, then outlet cells copy their x-1
    // neighbour, right to left; the host checked that no outlet cell starts a pack)
    uint32_t fl_any = 0u;
#pragma unroll
    for (int j = 0; j < V; ++j)
        fl_any |= 1u << (c[j] & CLS_FLAG);
    if (fl_any & ((1u << 3) | (1u << 4))) {
        if ((fl_any & (1u << 4)) && (fl_any & ((1u << 1) | (1u << 2)))) {
            // an outlet cell may copy from a wall cell: the wall's own (untouched) values
#pragma unroll
            for (int i = 0; i < Q; ++i) {
                T o[V];
                PackIO<TS, V>::load(a.f[i] + d, o);
#pragma unroll
                for (int j = 0; j < V; ++j)
                    if (!aa_participant(c[j]))
                        g[i][j] = o[j];
            }
        }
#pragma unroll
        for (int j = 0; j < V; ++j)
            if ((c[j] & CLS_FLAG) == 3) {
#pragma unroll
                for (int i = 0; i < Q; ++i)
                    g[i][j] = Store<TS>::up(a.inlet[i]);
            }
#pragma unroll
        for (int j = V - 1; j >= 1; --j)
            if ((c[j] & CLS_FLAG) == 4) {
#pragma unroll
                for (int i = 0; i < Q; ++i)
                    g[i][j] = g[i][j - 1];
            }
    }

    // ---- row-block layout: what crosses a warp boundary goes through shared memory
    int wr = -1, wl = -1;          // the warps holding the packs right / left of this warp's row
    __shared__ T pub0[ROWB ? 4 : 1][5], pub31[ROWB ? 4 : 1][5];
    __shared__ int pb0[ROWB ? 4 : 1], pb31[ROWB ? 4 : 1];
    if constexpr (ROWB) {
        if (lane == 0) {
            pb0[warp] = (int)bulk;
            int n = 0;
#define MLB_X(i, CX, Z, R) if (CX > 0) pub0[warp][n++] = g[opp(i)][0];
            MLB_DIRS(MLB_X)
#undef MLB_X
        }
        if (lane == 31) {
            pb31[warp] = (int)bulk;
            int n = 0;
#define MLB_X(i, CX, Z, R) if (CX < 0) pub31[warp][n++] = g[opp(i)][V - 1];
            MLB_DIRS(MLB_X)
#undef MLB_X
        }
        __syncthreads();
        // a block that spans the whole row closes it on itself (periodic wrap in x)
        const bool full = gridDim.x == 1 && gm.nx == WPR * 32 * V;
        wr = (wseg + 1 < WPR) ? warp + 1 : (full ? warp + 1 - WPR : -1);
        wl = (wseg > 0) ? warp - 1 : (full ? warp - 1 + WPR : -1);
        if (lane == 31)
            bulk_r = valid && wr >= 0 && pb0[wr] != 0 && (x0 + V < gm.nx || full);
        if (lane == 0)
            bulk_l = valid && wl >= 0 && pb31[wl] != 0;
    }

    // ---- stores ---------------------------------------------------------------
#define MLB_T(i, Z, R, X) aa_target<TS, CZ_##Z, REMOTE>(a, i, (Z), (R), (X), rlo, rhi)
    // The stores go to the very addresses the loads came from; left alone the
    // compiler keeps all 29 64-bit addresses alive across the collide (58
    // registers, which cost a resident block).  Laundering the 32-bit offsets
    // through an empty asm makes it rebuild them - one IMAD.WIDE each.
    int x0s = x0, xls = xl, xrs = xr, ds = d, zcs = zc, zms = zm, zqs = zq, rcs = rc, rms = rm,
        rqs = rq;
    asm volatile("" : "+r"(x0s), "+r"(xls), "+r"(xrs), "+r"(ds), "+r"(zcs), "+r"(zms), "+r"(zqs),
                      "+r"(rcs), "+r"(rms), "+r"(rqs));
    {
    const int x0 = x0s, xl = xls, xr = xrs, d = ds, zc = zcs, zm = zms, zq = zqs, rc = rcs,
              rm = rms, rq = rqs;
    (void)zc; (void)rc;
    // Bulk packs (no link bounces, every target location has this one writer):
    // aligned packs wherever the neighbouring lane can supply (or take) the
    // cell that crosses the pack boundary.  Directions are handled in three
    // groups (c_x = +1, -1, 0) so that only five shuffled values are live at a
    // time; every lane of the warp takes part in the shuffles.
    {
        T nb[5];
        int n = 0;
#define MLB_X(i, CX, Z, R) if (CX > 0) nb[n++] = __shfl_down_sync(FULL, g[opp(i)][0], 1);
        MLB_DIRS(MLB_X)
#undef MLB_X
        if constexpr (ROWB) {
            if (lane == 31 && wr >= 0) {
#pragma unroll
                for (int q = 0; q < 5; ++q) nb[q] = pub0[wr][q];
            }
        }
        if (bulk) {
            n = 0;
#define MLB_X(i, CX, Z, R)                                                            \
            if (CX > 0) { /* locations x0 .. x0+V-1 take cells x0+1 .. x0+V */        \
                /* straight-line, predicated stores: the lanes at the ends of a warp */ \
                /* row must not send the whole warp through a second code path       */ \
                TS *base = MLB_T(i, Z, R, x0);                                        \
                T o[V];                                                               \
                _Pragma("unroll") for (int j = 0; j < V - 1; ++j) o[j] = g[opp(i)][j + 1]; \
                o[V - 1] = nb[n];                                                     \
                PackIO<TS, V>::store_head(base, o, bulk_r);                           \
                { const TS v0 = Store<TS>::down(g[opp(i)][0]);                        \
                  if (!bulk_l) *MLB_T(i, Z, R, xl) = v0; }                            \
                ++n;                                                                  \
            }
            MLB_DIRS(MLB_X)
#undef MLB_X
        }
        n = 0;
#define MLB_X(i, CX, Z, R) if (CX < 0) nb[n++] = __shfl_up_sync(FULL, g[opp(i)][V - 1], 1);
        MLB_DIRS(MLB_X)
#undef MLB_X
        if constexpr (ROWB) {
            if (lane == 0 && wl >= 0) {
#pragma unroll
                for (int q = 0; q < 5; ++q) nb[q] = pub31[wl][q];
            }
        }
        if (bulk) {
            n = 0;
#define MLB_X(i, CX, Z, R)                                                            \
            if (CX < 0) { /* locations x0 .. x0+V-1 take cells x0-1 .. x0+V-2 */      \
                TS *base = MLB_T(i, Z, R, x0);                                        \
                T o[V];                                                               \
                _Pragma("unroll") for (int j = 1; j < V; ++j) o[j] = g[opp(i)][j - 1]; \
                o[0] = nb[n];                                                         \
                PackIO<TS, V>::store_tail(base, o, bulk_l);                           \
                { const TS v1 = Store<TS>::down(g[opp(i)][V - 1]);                    \
                  if (!bulk_r) *MLB_T(i, Z, R, xr) = v1; }                            \
                ++n;                                                                  \
            }
            MLB_DIRS(MLB_X)
#undef MLB_X
            PackIO<TS, V>::store(a.f[0] + d, g[0]);
#define MLB_X(i, CX, Z, R)                                                            \
            if (CX == 0)                                                              \
                PackIO<TS, V>::store(MLB_T(i, Z, R, x0), g[opp(i)]);
            MLB_DIRS(MLB_X)
#undef MLB_X
            return;
        }
    }
    if (!valid)
        return;
    // a pack with walls (or next to one): per cell, the scalar kernel's rules -
    // the result for opp(i) goes into the location read for i, or - bouncing
    // link - stays in the cell's own slot of opp(i) (kernels.py:88-96 read that)
#pragma unroll
    for (int j = 0; j < V; ++j)
        if (aa_participant(c[j]))
            a.f[0][d + j] = Store<TS>::down(g[0][j]);
#define MLB_X(i, CX, Z, R)                                                            \
    _Pragma("unroll") for (int j = 0; j < V; ++j)                                     \
        if (aa_participant(c[j])) {                                                   \
            const int xs = (CX) == 0 ? x0 + j                                         \
                         : (CX) > 0 ? (j == 0 ? xl : x0 + j - 1)                      \
                                    : (x0 + j + 1 >= gm.nx ? 0 : x0 + j + 1);         \
            if (c[j] & cls_link(i)) a.f[opp(i)][d + j] = Store<TS>::down(g[opp(i)][j]); \
            else *MLB_T(i, Z, R, xs) = Store<TS>::down(g[opp(i)][j]);                 \
        }
    MLB_DIRS(MLB_X)
#undef MLB_X
#undef MLB_T
    }
}

// aa_local_vec_kernel (R1 -> R0): everything a cell needs is in its own slots.
template <typename TS, int V, int LX, bool PUSH>
__global__ void __launch_bounds__(128, 4) aa_local_vec_kernel(const AAArgs<TS> a,
                                                              const PushArgs<TS> ph)
{
    using T = typename Store<TS>::C;
    constexpr int RPW = 32 / LX;
    const Geom &gm = a.g;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int x0 = (blockIdx.x * LX + (lane % LX)) * V;
    const int y = blockIdx.y * (4 * RPW) + warp * RPW + lane / LX;
    // the row padding is rewritten too (always valid in place): whole last lines
    if (x0 >= (int)gm.xp || y >= gm.ny)
        return;
    const int lz = a.z0 + (int)blockIdx.z;
    const int d = (lz + 1) * (int)gm.plane + y * (int)gm.xp + x0;

    const uint32_t kpack = KindIO<V>::load(a.ct.kind + d);
    T g[Q][V];
#pragma unroll
    for (int i = 0; i < Q; ++i)
        PackIO<TS, V>::load(a.f[opp(i)] + d, g[i]);
    if (a.pf_bulk) {
        if (blockIdx.x == 0 && threadIdx.x < Q && (a.pf_dz | a.pf_dy) != 0)
            prefetch_rows<TS, false>(a.f, gm, a.pf_dz, a.pf_dy, blockIdx.y * (4 * RPW), 4 * RPW, lz,
                                     threadIdx.x);
    } else
        prefetch_ahead<TS, V, LX, false>(a.f, gm, a.pf_dz, a.pf_dy, x0, y, lz, lane);
    uint32_t c[V];
#pragma unroll
    for (int j = 0; j < V; ++j)
        c[j] = 0u;
    if (kpack != 0u) {
#pragma unroll
        for (int j = 0; j < V; ++j) {
            const uint32_t k = (kpack >> (8 * j)) & 0xffu;
            if (k != 0u)
                c[j] = cls_of(a.ct, k, d + j);
        }
        // a bounced population still lacks its moving-wall term
#pragma unroll
        for (int j = 0; j < V; ++j)
            if ((c[j] & CLS_FLAG) == 0 && (c[j] & CLS_MOVING)) {
                const uint32_t mv = mlinks_of(a.ct, (kpack >> (8 * j)) & 0xffu, d + j);
#pragma unroll
                for (int i = 1; i < Q; ++i)
                    if (mv & (1u << i))
                        g[i][j] = g[i][j] + a.k[i];
            }
    }
    if constexpr (UsePackedMath<TS>::value)
        collide_cell_pairs<V>(g, a.omega);
    else
        collide_cells<T, V>(g, a.omega);
    bool allfluid = true;
#pragma unroll
    for (int j = 0; j < V; ++j)
        allfluid &= (c[j] & CLS_FLAG) == 0;
    if (!allfluid) {
        // wall cells keep their (still unmodified) values: full-line stores
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            T o[V];
            PackIO<TS, V>::load(a.f[i] + d, o);
#pragma unroll
            for (int j = 0; j < V; ++j)
                if ((c[j] & CLS_FLAG) != 0)
                    g[i][j] = o[j];
        }
        // open-boundary cells: new state by rule (see aa_pull_vec_kernel)
#pragma unroll
        for (int j = 0; j < V; ++j)
            if ((c[j] & CLS_FLAG) == 3) {
#pragma unroll
                for (int i = 0; i < Q; ++i)
                    g[i][j] = Store<TS>::up(a.inlet[i]);
            }
#pragma unroll
        for (int j = V - 1; j >= 1; --j)
            if ((c[j] & CLS_FLAG) == 4) {
#pragma unroll
                for (int i = 0; i < Q; ++i)
                    g[i][j] = g[i][j - 1];
            }
    }
#pragma unroll
    for (int i = 0; i < Q; ++i)
        PackIO<TS, V>::store(a.f[i] + d, g[i]);
    if constexpr (PUSH) {
        // z-slabs: the block is back in the normal representation; the crossing
        // populations of a boundary plane also go into the ring neighbour's halo
        // plane, exactly as in the two-buffer kernel (full packs: the halo of a
        // wall cell then holds the wall's own values, which nobody reads)
        const int o = y * (int)gm.xp + x0;
        if (lz == 0 && ph.lo[0] != nullptr) {
#pragma unroll
            for (int j = 0; j < 5; ++j)
                PackIO<TS, V>::store(ph.lo[j] + o, g[halo_down(j)]);
        }
        if (lz == gm.nz - 1 && ph.hi[0] != nullptr) {
#pragma unroll
            for (int j = 0; j < 5; ++j)
                PackIO<TS, V>::store(ph.hi[j] + o, g[halo_up(j)]);
        }
    }
}

// ---------------------------------------------------------------------------
// Class words (and the moving-wall link bits) from the padded flag block,
// halo planes already filled.  One thread per padded element of storage
// planes [0, nz+2).  Direction i's source is the neighbour at -c_i, with the
// same periodic wrap / halo-plane rule as the step kernels.
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

// class word + moving-wall link bits of one padded element of the flag block
__device__ __forceinline__ void cell_class(const uint8_t *__restrict__ flags, const Geom &gm,
                                           int x, int y, int sz, uint32_t &cw, uint32_t &mw)
{
    const long long d = (long long)sz * gm.plane + (long long)y * gm.xp + x;
    mw = 0u;
    if (x >= gm.nx) {
        cw = 1u;  // row padding: solid, never written
        return;
    }
    const uint32_t fl = flags[d];
    if (sz == 0 || sz == gm.nz + 1 || fl == 1 || fl == 2) {
        cw = fl;  // halo planes are only ever sources; walls have no links
        return;
    }
    // fluid cells - and inlet / outlet cells, whose link bits only the in-place
    // kernels look at (there every non-wall cell takes part in the exchange)
    const int lz = sz - 1;
    // index 0: same, 1: the "minus" neighbour (source for c = +1), 2: the "plus" one
    const int xs[3] = {x, (x == 0) ? gm.nx - 1 : x - 1, (x == gm.nx - 1) ? 0 : x + 1};
    const int ys[3] = {y, (y == 0) ? gm.ny - 1 : y - 1, (y == gm.ny - 1) ? 0 : y + 1};
    const int zs[3] = {sz, (lz == 0) ? gm.zlo_src : lz, (lz == gm.nz - 1) ? gm.zhi_src : lz + 2};
    const int cof[3] = {0, 1, -1};  // the c component served by index 0/1/2
    uint32_t c = 0u, mv = 0u;
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
                    c |= cls_link(i);
                if (m == 2)
                    mv |= 1u << i;
            }
    cw = fl | c | (mv ? CLS_MOVING : 0u);
    mw = mv;
}

// Census of the padded flag block: [0] inlet cells, [1] outlet cells (slab
// planes only), [2] unknown codes (anywhere, halo planes included).
__global__ void flag_census_kernel(const uint8_t *__restrict__ flags, const Geom gm,
                                   unsigned long long *__restrict__ out)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    const int sz = blockIdx.z;
    uint8_t m = 0;
    if (x < gm.nx)
        m = flags[(long long)sz * gm.plane + (long long)blockIdx.y * gm.xp + x];
    const bool interior = sz >= 1 && sz <= gm.nz;
    const unsigned b3 = __ballot_sync(0xffffffffu, interior && m == 3);
    const unsigned b4 = __ballot_sync(0xffffffffu, interior && m == 4);
    const unsigned bx = __ballot_sync(0xffffffffu, m > 4);
    if ((threadIdx.x & 31) == 0) {
        if (b3) atomicAdd(&out[0], (unsigned long long)__popc(b3));
        if (b4) atomicAdd(&out[1], (unsigned long long)__popc(b4));
        if (bx) atomicAdd(&out[2], (unsigned long long)__popc(bx));
    }
}

// The dictionary: every distinct (class word, link bits) pair gets a slot of a
// 256-entry open-addressing table (slot 0 = the bulk pair (0, 0), slot 255 =
// escape, never a key); kind[d] = the slot.  Slot numbers depend on insertion
// order, which no result depends on.
constexpr unsigned long long KIND_EMPTY = ~0ull;
// One pass from the flags to the kind bytes: the class word of a cell lives in
// registers only.  cls_full / ml_full are NULL on the first pass; if the
// dictionary overflowed (escapes > 0) the host allocates them and runs the pass
// again - the table is then full, so every cell finds its old slot or escapes -
// and the escape cells get their full-width words.
__global__ void build_kind_kernel(const uint8_t *__restrict__ flags, const Geom gm,
                                  unsigned long long *__restrict__ tab, uint8_t *__restrict__ kind,
                                  unsigned int *__restrict__ escapes,
                                  uint32_t *__restrict__ cls_full, uint32_t *__restrict__ ml_full)
{
    const int x = blockIdx.x * blockDim.x + threadIdx.x;
    if (x >= gm.xp)
        return;
    const int y = blockIdx.y, sz = blockIdx.z;  // storage plane
    const long long d = (long long)sz * gm.plane + (long long)y * gm.xp + x;
    uint32_t cw, mw;
    cell_class(flags, gm, x, y, sz, cw, mw);
    const unsigned long long key = ((unsigned long long)mw << 32) | cw;
    if (key == 0ull) {
        kind[d] = 0;
        return;
    }
    unsigned int h = (unsigned int)((key * 0x9E3779B97F4A7C15ull) >> 40);
    for (int probe = 0; probe < 254; ++probe) {
        const unsigned int s = 1u + (h + probe) % 254u;  // 1..254
        const unsigned long long old = atomicCAS(&tab[s], KIND_EMPTY, key);
        if (old == KIND_EMPTY || old == key) {
            kind[d] = (uint8_t)s;
            return;
        }
    }
    kind[d] = (uint8_t)KIND_ESCAPE;
    atomicAdd(escapes, 1u);
    if (cls_full) {
        cls_full[d] = cw;
        ml_full[d] = mw;
    }
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
template <typename T, bool INCELL = false>
__device__ __forceinline__ void cell_moments(const T *__restrict__ f, long long d,
                                             long long pop, double &r, double &mx,
                                             double &my, double &mz, int *bad)
{
    double v[Q];
#pragma unroll
    for (int i = 0; i < Q; ++i) {
        v[i] = (double)Store<T>::up(f[(long long)i * pop + d]);
        if (!INCELL && bad && !isfinite(v[i]))
            ++*bad;
    }
    r = v[0];
#pragma unroll
    for (int i = 1; i < Q; ++i)
        r = r + v[i];
    // INCELL: the values are tested only where the cell's sum is non-finite, and re-read
    // for it (cache hits, and rare) rather than kept in registers - see diag_kernel
    if (INCELL && bad && !isfinite(r)) {
#pragma unroll 1
        for (int i = 0; i < Q; ++i)
            if (!isfinite((double)Store<T>::up(f[(long long)i * pop + d])))
                ++*bad;
    }
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

// Pack forms of the two diagnostics kernels: V consecutive cells per thread,
// all 19 pack loads issued together (16-byte words in fp32 / fp64, 8 bytes
// with fp16 storage), moments accumulated in float64 in the SAME left-to-right
// order as cell_moments - the terms of rho, m_x, m_y, m_z all appear in
// increasing population order - so every value is bit-identical to the
// one-cell-per-thread kernels (and the oracle).
template <typename TS, int V>
__device__ __forceinline__ void pack_moments(const TS *__restrict__ f, long long d, long long pop,
                                             double (&r)[V], double (&mx)[V], double (&my)[V],
                                             double (&mz)[V], int *bad)
{
    using T = typename Store<TS>::C;
    T w[Q][V];
#pragma unroll
    for (int i = 0; i < Q; ++i)
        PackIO<TS, V>::load(f + (long long)i * pop + d, w[i]);
#pragma unroll
    for (int j = 0; j < V; ++j) {
        double v[Q];
#pragma unroll
        for (int i = 0; i < Q; ++i) {
            v[i] = (double)w[i][j];
            if (bad && !isfinite(w[i][j]))
                ++*bad;
        }
        double t = v[0];
#pragma unroll
        for (int i = 1; i < Q; ++i)
            t = t + v[i];
        r[j] = t;
        mx[j] = v[1] - v[3] + v[5] - v[6] - v[7] + v[8] + v[11] - v[12] - v[13] + v[14];
        my[j] = v[2] - v[4] + v[5] + v[6] - v[7] - v[8] + v[15] - v[16] - v[17] + v[18];
        mz[j] = v[9] - v[10] + v[11] + v[12] - v[13] - v[14] + v[15] + v[16] - v[17] - v[18];
    }
}

template <int V>
__device__ __forceinline__ void store_doubles(double *p, const double (&v)[V])
{
#pragma unroll
    for (int j = 0; j < V; j += 2)
        *reinterpret_cast<double2 *>(p + j) = make_double2(v[j], v[j + 1]);
}

template <typename TS, int V>
__global__ void __launch_bounds__(128)
macro_vec_kernel(const TS *__restrict__ f, const Geom gm, double *__restrict__ rho,
                 double *__restrict__ ux, double *__restrict__ uy, double *__restrict__ uz)
{
    const int x0 = (blockIdx.x * 128 + threadIdx.x) * V;
    if (x0 >= gm.nx)
        return;
    const int y = blockIdx.y, lz = blockIdx.z;
    const long long d = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp + x0;
    const long long o = ((long long)lz * gm.ny + y) * gm.nx + x0;
    double r[V], mx[V], my[V], mz[V];
    pack_moments<TS, V>(f, d, gm.pop, r, mx, my, mz, nullptr);
    double a[V], b[V], c[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        a[j] = (r[j] != 0.0) ? mx[j] / r[j] : 0.0;
        b[j] = (r[j] != 0.0) ? my[j] / r[j] : 0.0;
        c[j] = (r[j] != 0.0) ? mz[j] / r[j] : 0.0;
    }
    store_doubles<V>(rho + o, r);
    store_doubles<V>(ux + o, a);
    store_doubles<V>(uy + o, b);
    store_doubles<V>(uz + o, c);
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

// LAZY: how non-finite VALUES are counted.  0: every value is tested as it is converted.
// 1: only a thread whose mass sum says it met one counts - a NaN or an infinity among the
// terms makes every later partial sum non-finite (the converse, finite float64 terms
// overflowing, takes the exact count and finds none) - by walking its cells again after
// the loop; the common case then pays nothing per value.  2 (one cell per thread only):
// the same test per cell, on the cell's own sum.  All give the same count; which one an
// instantiation uses was chosen by measurement (removing the per-value tests changes the
// register allocation, and with it how many loads the compiler keeps in flight).
template <typename T, int LAZY>
__global__ void __launch_bounds__(DIAG_THREADS)
diag_kernel(const T *__restrict__ f, const ClsTab ct, const Geom gm,
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
            if (LAZY == 1)
                cell_moments<T>(f, d, gm.pop, rr, mx, my, mz, nullptr);
            else
                cell_moments<T, LAZY == 2>(f, d, gm.pop, rr, mx, my, mz, &bad);
            acc[0] += rr;
            acc[6] += (double)bad;
            const uint32_t kd = ct.kind[d];
            if (kd == 0 || (cls_of(ct, kd, (int)d) & CLS_FLAG) == 0) {
                acc[7] += 1.0;
                acc[1] += mx;
                acc[2] += my;
                acc[3] += mz;
                if (rr != 0.0) {
                    const double u2 = (mx * mx + my * my + mz * mz) / (rr * rr);
                    acc[4] += 0.5 * rr * u2;
                    acc[5] = fmax(acc[5], u2);  // max |u|^2; the root is taken once, at the end
                }
            }
        }
    }
    if (LAZY == 1 && !isfinite(acc[0])) {
        int bad = 0;
        for (long long r = blockIdx.x; r < rows; r += gridDim.x) {
            const int lz = (int)(r / gm.ny), y = (int)(r % gm.ny);
            const long long base = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp;
            for (int x = threadIdx.x; x < gm.nx; x += DIAG_THREADS)
#pragma unroll 1
                for (int i = 0; i < Q; ++i)
                    if (!isfinite((double)Store<T>::up(f[(long long)i * gm.pop + base + x])))
                        ++bad;
        }
        acc[6] = (double)bad;  // (0 so far)
    }
    diag_block_reduce(acc, partials + (long long)blockIdx.x * DIAG_N);
}

// pack form: a fixed assignment of packs to threads, cells of a pack in order
template <typename TS, int V, bool LAZY>
__global__ void __launch_bounds__(DIAG_THREADS)
diag_vec_kernel(const TS *__restrict__ f, const ClsTab ct, const Geom gm,
                double *__restrict__ partials)
{
    double acc[DIAG_N];
#pragma unroll
    for (int i = 0; i < DIAG_N; ++i)
        acc[i] = 0.0;
    // a block works on `rpi` rows per iteration: thread t owns pack t % ppr of
    // sub-row t / ppr (short rows), or packs t, t + 256, ... of one row (long rows)
    const int ppr = gm.nx / V;  // packs per row
    const int rpi = ppr >= DIAG_THREADS ? 1 : DIAG_THREADS / ppr;
    const int sub = ppr >= DIAG_THREADS ? 0 : (int)threadIdx.x / ppr;
    const int pk0 = ppr >= DIAG_THREADS ? (int)threadIdx.x : (int)threadIdx.x - sub * ppr;
    const long long rows = (long long)gm.nz * gm.ny;
    for (long long row = (long long)blockIdx.x * rpi + sub; sub < rpi && row < rows;
         row += (long long)gridDim.x * rpi) {
        const int lz = (int)(row / gm.ny), y = (int)(row - (long long)lz * gm.ny);
        for (int x0 = pk0 * V; x0 < gm.nx; x0 += DIAG_THREADS * V) {
            const long long d = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp + x0;
            const uint32_t kpack = KindIO<V>::load(ct.kind + d);
            double rr[V], mx[V], my[V], mz[V];
            int bad = 0;
            if (LAZY)
                pack_moments<TS, V>(f, d, gm.pop, rr, mx, my, mz, nullptr);
            else
                pack_moments<TS, V>(f, d, gm.pop, rr, mx, my, mz, &bad);
            acc[6] += (double)bad;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                acc[0] += rr[j];
                const uint32_t kd = (kpack >> (8 * j)) & 0xffu;
                if (kd == 0 || (cls_of(ct, kd, (int)d + j) & CLS_FLAG) == 0) {
                    acc[7] += 1.0;
                    acc[1] += mx[j];
                    acc[2] += my[j];
                    acc[3] += mz[j];
                    if (rr[j] != 0.0) {
                        const double u2 = (mx[j] * mx[j] + my[j] * my[j] + mz[j] * mz[j])
                                          / (rr[j] * rr[j]);
                        acc[4] += 0.5 * rr[j] * u2;
                        acc[5] = fmax(acc[5], u2);
                    }
                }
            }
        }
    }
    if (LAZY && !isfinite(acc[0])) {  // see diag_kernel: the exact count, only where the sum asks for it
        using T = typename Store<TS>::C;
        int bad = 0;
        for (long long row = (long long)blockIdx.x * rpi + sub; sub < rpi && row < rows;
             row += (long long)gridDim.x * rpi) {
            const int lz = (int)(row / gm.ny), y = (int)(row - (long long)lz * gm.ny);
            for (int x0 = pk0 * V; x0 < gm.nx; x0 += DIAG_THREADS * V) {
                const long long d = (long long)(lz + 1) * gm.plane + (long long)y * gm.xp + x0;
#pragma unroll 1
                for (int i = 0; i < Q; ++i) {
                    T w[V];
                    PackIO<TS, V>::load(f + (long long)i * gm.pop + d, w);
#pragma unroll
                    for (int j = 0; j < V; ++j)
                        if (!isfinite(w[j]))
                            ++bad;
                }
            }
        }
        acc[6] = (double)bad;  // (0 so far)
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
    // the kernels track max |u|^2: sqrt is monotone and correctly rounded, so the
    // root of the maximum is the maximum of the roots
    if (threadIdx.x == 0)
        out[5] = sqrt(out[5]);
}

}  // namespace mlb
