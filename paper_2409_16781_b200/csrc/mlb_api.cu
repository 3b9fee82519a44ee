// mlb_api.cu - host side of the C ABI declared in include/mlb.h.
//
// Thin: argument checks, the flag-derived tables, launches.  All device
// code lives in mlb_kernels.cuh.  Build (see csrc/Makefile):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -fmad=false
//        -shared -Xcompiler -fPIC -o libmlb_d3q19.so mlb_api.cu
#include "../../include/mlb.h"
#include "mlb_kernels.cuh"

#include <atomic>
#include <chrono>
#include <map>
#include <mutex>
#include <unordered_map>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <type_traits>
#include <vector>

namespace {

thread_local char g_err[512] = "";
std::atomic<long long> g_launches{0};

int fail(int code, const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

#define MLB_CUDA(expr)                                                          \
    do {                                                                        \
        cudaError_t e_ = (expr);                                                \
        if (e_ != cudaSuccess)                                                  \
            return fail(MLB_ECUDA, "%s: %s (%s:%d)", #expr,                     \
                        cudaGetErrorString(e_), __FILE__, __LINE__);            \
    } while (0)

#define MLB_LAUNCHED()                                                          \
    do {                                                                        \
        g_launches.fetch_add(1, std::memory_order_relaxed);                     \
        MLB_CUDA(cudaGetLastError());                                           \
    } while (0)

inline cudaStream_t S(void *s) { return static_cast<cudaStream_t>(s); }

// Entry points work on the plan's device and leave the caller's current device
// as they found it (a process may drive several GPUs, or keep torch's current
// device elsewhere).
struct DeviceGuard {
    int prev = -1;
    bool switched = false;
    cudaError_t err = cudaSuccess;
    explicit DeviceGuard(int dev)
    {
        err = cudaGetDevice(&prev);
        if (err == cudaSuccess && prev != dev) {
            err = cudaSetDevice(dev);
            switched = err == cudaSuccess;
        }
    }
    ~DeviceGuard()
    {
        if (switched)
            cudaSetDevice(prev);
    }
    DeviceGuard(const DeviceGuard &) = delete;
    DeviceGuard &operator=(const DeviceGuard &) = delete;
};
#define MLB_ON_DEVICE(dev)                                                      \
    DeviceGuard guard_(dev);                                                    \
    if (guard_.err != cudaSuccess)                                              \
        return fail(MLB_ECUDA, "cudaSetDevice(%d): %s", (int)(dev),             \
                    cudaGetErrorString(guard_.err))

// Device memory of the plans (flag tables, index lists, reduction scratch, signal
// words) comes from a small process-wide pool: cudaMalloc / cudaFree synchronise
// the device and were measured to stall for 0.1 - 1.4 s now and then with tens of
// GB of populations resident - a large, erratic part of a short run's end-to-end
// time (plan setup + teardown are inside engine.run).  Freed blocks are kept,
// keyed by (device, size), and handed out again to the next plan of the same
// shape; at most POOL_CAP bytes are held back, mlb_trim() returns them all.
class DevicePool {
public:
    explicit DevicePool(size_t cap) : cap_(cap) {}
    cudaError_t alloc(void **out, size_t bytes)
    {
        int dev = 0;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> g(mu_);
            auto it = free_.find({dev, bytes});
            if (it != free_.end()) {
                *out = it->second;
                free_.erase(it);
                cached_ -= bytes;
                live_[*out] = {dev, bytes};
                return cudaSuccess;
            }
        }
        cudaError_t e = cudaMalloc(out, bytes);
        if (e != cudaSuccess) {       // give the pool's idle memory back and retry once
            trim();
            e = cudaMalloc(out, bytes);
        }
        if (e == cudaSuccess) {
            std::lock_guard<std::mutex> g(mu_);
            live_[*out] = {dev, bytes};
        }
        return e;
    }
    void release(void *p)
    {
        if (!p) return;
        std::lock_guard<std::mutex> g(mu_);
        auto it = live_.find(p);
        if (it == live_.end()) {      // not ours
            cudaFree(p);
            return;
        }
        const Key k = it->second;
        live_.erase(it);
        if (cached_ + k.second > cap_) {
            cudaFree(p);
            return;
        }
        free_.insert({k, p});
        cached_ += k.second;
    }
    void trim()
    {
        std::lock_guard<std::mutex> g(mu_);
        for (auto &kv : free_)
            cudaFree(kv.second);
        free_.clear();
        cached_ = 0;
    }

private:
    using Key = std::pair<int, size_t>;
    const size_t cap_;
    std::mutex mu_;
    std::multimap<Key, void *> free_;
    std::unordered_map<void *, Key> live_;
    size_t cached_ = 0;
};
DevicePool g_pool(6ull << 30);
// Population blocks handed out by mlb_block_alloc: plain cudaMalloc memory (what
// CUDA IPC can export, whatever allocator the host framework is configured with).
// A short run allocates and frees tens of GB around a few milliseconds of work,
// so up to MLB_BLOCK_POOL_GB (default 24) of freed blocks are kept for the next
// caller; an allocation that fails returns them to the driver and retries.
size_t block_pool_cap()
{
    const char *e = std::getenv("MLB_BLOCK_POOL_GB");
    const double gb = e ? std::atof(e) : 24.0;
    return gb <= 0.0 ? 0 : (size_t)(gb * (double)(1ull << 30));
}
DevicePool g_blocks(block_pool_cap());

template <typename T>
cudaError_t pool_alloc(T **out, size_t bytes) { return g_pool.alloc(reinterpret_cast<void **>(out), bytes); }
inline void pool_free(void *p) { g_pool.release(p); }

}  // namespace

struct mlb_plan {
    int nx = 0, ny = 0, nz = 0, dtype = 0, device = 0, z_mode = 0, variant = 0;
    int passthrough = 0;
    long long prefetch = -1;  // L2 prefetch distance in cells, -1 = auto (prefetch_distance)
    double omega = 1.0, wall_u[3] = {0, 0, 0}, inlet_u = 0.0;
    mlb_layout lay{};
    mlb::Geom g{};
    bool have_flags = false;
    uint8_t *d_flags = nullptr;  // padded flag block incl. halo planes
    // what the kernels read: one kind byte per cell (same shape as d_flags) + the
    // dictionary of distinct (class word, moving-wall link bits) pairs
    uint8_t *d_kind = nullptr;
    unsigned long long *d_tab = nullptr;  // [256]
    // full-width per-cell class words / link bits: scratch of the build, kept
    // only when the geometry has more than 254 distinct pairs (escape cells)
    uint32_t *d_cls = nullptr;
    uint32_t *d_mlinks = nullptr;
    unsigned int n_escape = 0, n_kinds = 0;
    // open-boundary index lists, sorted by (lz, y, x); *_zoff[lz] = first entry of plane lz
    long long n_in = 0, n_out = 0;
    long long *d_in = nullptr, *d_out = nullptr;
    std::vector<long long> in_zoff, out_zoff;
    bool out_chained = false;
    unsigned out_xmod8 = 0;  // bit r set: some outlet cell has x % 8 == r
    void *d_out_tmp = nullptr;
    // reductions
    int sms = 148;
    int diag_blocks = 0;
    double *d_partials = nullptr, *d_diag = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // bumped by every setter that changes what a launch looks like: a captured
    // graph of step launches is only replayed while it still matches
    unsigned long long epoch = 0;
    // CUDA graph of a run of steps (mlb_run_steps / mlb_run_steps_inplace on small,
    // launch-bound domains): captured once on the library's own stream, replayed on
    // the caller's
    int aa_layout = -1;             // in-place pull half: 1 = row-block layout, 0 / -1 = classic
    int graph_mode = -1;            // -1 auto (small domains), 0 never, 1 always
    cudaStream_t cap_stream = nullptr;
    struct GraphCache {
        cudaGraphExec_t exec = nullptr;
        void *a = nullptr, *b = nullptr;
        unsigned long long epoch = 0;
        int steps = 0, repr = 0;
        long long nodes = 0;
    } gc;
    // z-slab schedule (mlb_slab_run_steps): fork / join between the main and the
    // boundary stream
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    // host-resident runs (mlb_run_steps_host): planes 0 and nz-1 hold no fluid /
    // open-boundary cell, so no update depends on the periodic wrap in z and the
    // domain can be stepped chunk by chunk behind the upload
    bool z_closed = false;
    cudaStream_t up_stream = nullptr, down_stream = nullptr;
    unsigned int *d_work = nullptr;   // staged kernel: ring of work counters, one per launch
    unsigned int work_next = 0;
};

namespace {

int layout_of(int nx, int ny, int nz, int dtype, mlb_layout *out)
{
    if (nx < 1 || ny < 1 || nz < 1)
        return fail(MLB_EINVAL, "grid %dx%dx%d is empty", nx, ny, nz);
    if (dtype != MLB_F32 && dtype != MLB_F64 && dtype != MLB_F16 && dtype != MLB_F32C64)
        return fail(MLB_EINVAL, "unknown dtype code %d (0 = f32, 1 = f64, 2 = f16 storage / "
                    "f32 compute, 3 = f32 storage / f64 compute)", dtype);
    if (ny > 65535 || nz > 65535)
        return fail(MLB_EUNSUPPORTED, "ny and nz are limited to 65535 per slab");
    const int sz = dtype == MLB_F64 ? 8 : dtype == MLB_F16 ? 2 : 4;
    const long long line = 128 / sz;
    out->nx = nx; out->ny = ny; out->nz = nz; out->itemsize = sz;
    out->xp = (nx + line - 1) / line * line;
    out->plane = (long long)ny * out->xp;
    out->pop = (long long)(nz + 2) * out->plane;
    if (out->pop >= (1LL << 31))
        return fail(MLB_EUNSUPPORTED, "slab of %dx%dx%d cells exceeds 2^31 elements per "
                    "population; use more z-slabs", nx, ny, nz);
    out->total = MLB_Q * out->pop;
    out->bytes = out->total * sz;
    return MLB_OK;
}

void set_geom(mlb_plan *p)
{
    p->g.nx = p->nx; p->g.ny = p->ny; p->g.nz = p->nz;
    p->g.xp = p->lay.xp; p->g.plane = p->lay.plane; p->g.pop = p->lay.pop;
    if (p->z_mode == MLB_Z_PERIODIC) {
        p->g.zlo_src = p->nz;  // storage plane of lz = nz-1
        p->g.zhi_src = 1;      // storage plane of lz = 0
    } else {
        p->g.zlo_src = 0;
        p->g.zhi_src = p->nz + 1;
    }
}

mlb::ClsTab cls_tab(const mlb_plan *p)
{
    mlb::ClsTab t;
    t.kind = p->d_kind;
    t.tab = reinterpret_cast<const uint2 *>(p->d_tab);  // little-endian: x = class word, y = links
    t.cls_full = p->d_cls;
    t.ml_full = p->d_mlinks;
    return t;
}

template <typename T>
void wall_terms(const double *uw, T *k)
{
    // 6 w_i (c_i . u_w): one product per +direction, the opposite by
    // negation, as kernels.py:249-256 builds its eight.
    const T ms = T(1.0 / 3.0), md = T(1.0 / 6.0);
    const T x = T(uw[0]), y = T(uw[1]), z = T(uw[2]);
    k[0] = T(0.0);
    k[1] = ms * x;        k[3] = -k[1];
    k[2] = ms * y;        k[4] = -k[2];
    k[5] = md * (x + y);  k[7] = -k[5];
    k[6] = md * (y - x);  k[8] = -k[6];
    k[9] = ms * z;        k[10] = -k[9];
    k[11] = md * (x + z); k[13] = -k[11];
    k[12] = md * (z - x); k[14] = -k[12];
    k[15] = md * (y + z); k[17] = -k[15];
    k[16] = md * (z - y); k[18] = -k[16];
}

// equilibrium(1, u_in, 0, 0) in compute dtype, lattice.py:60-109 factoring.
// Host code: the Makefile passes -ffp-contract=off to the host compiler so
// this is one rounding per operation, like the device code.
template <typename T>
void inlet_values(double u_in, T *e)
{
    const T one = T(1.0), c3 = T(3.0), c45 = T(4.5), c15 = T(1.5);
    const T w0 = T(1.0 / 3.0), ws = T(1.0 / 18.0), wd = T(1.0 / 36.0);
    const T rho = T(1.0), ux = T(u_in), uy = T(0.0), uz = T(0.0);
    const T usq = ux * ux + uy * uy + uz * uz;
    const T um = one - c15 * usq;
    const T wr0 = w0 * rho, wrs = ws * rho, wrd = wd * rho;
    auto pair = [&](T cu, T wr, int ip, int im) {
        const T q = c45 * (cu * cu);
        const T t = c3 * cu;
        const T p = um + q;
        e[ip] = wr * (p + t);
        e[im] = wr * (p - t);
    };
    pair(ux, wrs, 1, 3);
    pair(uy, wrs, 2, 4);
    pair(ux + uy, wrd, 5, 7);
    pair(ux - uy, wrd, 8, 6);
    pair(uz, wrs, 9, 10);
    pair(ux + uz, wrd, 11, 13);
    pair(ux - uz, wrd, 14, 12);
    pair(uy + uz, wrd, 15, 17);
    pair(uy - uz, wrd, 18, 16);
    e[0] = wr0 * um;
}

// Kernel variants (mlb_plan_set_variant).  0 = auto; 32..512 = one cell per
// thread with that block width; W * 1000 + LX = packs of (16 >> (W - 1)) bytes
// (W = 1: 16 B = 4 floats / 2 doubles; W = 2: 8 B = 4 halves; W = 3: 4 B =
// 2 halves) with LX = 8 / 16 / 32 packs per warp row.
constexpr int VARIANT_STAGED = 4000;   // step_stage_kernel: rows staged through shared memory

int pack_cells(int dtype, int variant)
{
    if (variant == VARIANT_STAGED)   // 16-byte packs, 8 bytes with fp16 / fp32-for-fp64 storage
        return dtype == MLB_F32 ? 4 : dtype == MLB_F16 ? 4 : 2;
    const int bytes = 16 >> (variant / 1000 - 1);
    const int sz = dtype == MLB_F64 ? 8 : dtype == MLB_F16 ? 2 : 4;
    return bytes / sz;
}

bool variant_exists(int dtype, int variant)
{
    if (variant == 0 || variant == 32 || variant == 64 || variant == 128 || variant == 256
        || variant == 512 || variant == VARIANT_STAGED)
        return true;
    const int w = variant / 1000, lx = variant % 1000;
    if (lx != 8 && lx != 16 && lx != 32)
        return false;
    if (dtype == MLB_F16)
        return w == 2 || w == 3;
    if (dtype == MLB_F32C64)
        return w == 2;   // 8-byte packs: two floats, two doubles' worth of registers per population
    if (dtype == MLB_F32)
        return w == 1 || w == 2;   // 16-byte packs, or 8-byte packs (even rows that 4 does not divide)
    return w == 1;
}

// The staged kernel (step_stage_kernel): a warp per column of 32 packs; it serves
// any row length (ragged rows and the periodic wrap are index arithmetic inside
// the staged segment) as long as a block's staging buffers fit shared memory.
template <typename TS, int V>
constexpr size_t stage_smem() { return 4 * (size_t)mlb::StageShape<TS, V>::WARP_BYTES; }
bool stage_shape(const mlb_plan *p)
{
    // fp16 storage and fp32 storage / fp64 arithmetic (see StageShape::OK)
    return (p->dtype == MLB_F16 || p->dtype == MLB_F32C64) && p->nx >= 2;
}

// the kernel `variant` resolves to for this plan (0 = auto); measured on B200
// with tools/sweep.py: packs win in fp32 and fp16 storage, not in fp64
int resolve_variant(const mlb_plan *p, bool allow_staged = true)
{
    const bool special = p->variant == VARIANT_STAGED;
    if (p->variant != 0 && !(special && !allow_staged)) {
        if (!special || stage_shape(p))
            return p->variant;
    }
    // fp32 and fp16 storage: packs of four cells for any row length - a row the pack
    // does not divide ends in a pack of real cells + padding (511^3, fraction of the HBM
    // peak: fp32 0.984 one cell per thread -> 1.002 packs; fp16 storage 0.62 -> see DESIGN)
    static const int ragged = std::getenv("MLB_RAGGED_PACKS") ? std::atoi(std::getenv("MLB_RAGGED_PACKS")) : 1;
    if (p->dtype == MLB_F32 && (p->nx % 4 == 0 || ragged) && p->nx >= 128)
        return 1016;
    if (p->dtype == MLB_F16 && (p->nx % 4 == 0 || ragged) && p->nx >= 128)
        return 2008;
    // fp64: the scalar kernel is ~2 % faster, unless there are open-boundary
    // cells, which only a pack kernel can handle inside the fused pass (~7 %)
    if (p->dtype == MLB_F64 && (p->n_in || p->n_out) && p->nx % 2 == 0 && p->nx >= 128)
        return 1016;
    if (p->dtype == MLB_F32C64 && p->nx % 2 == 0 && p->nx >= 128)
        return 2016;   // 8-byte packs: 36.6 vs 33.4 GLUPS (one cell per thread) at 512^3.  (With its
                       // bulk L2 prefetch the one-cell-per-thread kernel is 3 % ahead in 200-step
                       // runs - 0.936 vs 0.907 of the HBM peak - but 1 % behind in the 300-step
                       // bench at the power cap, 37.9 vs 38.2 GLUPS: packs stay the default.)
    return 128;
}

template <typename T>
void inlet_values(double u_in, T *e);

// can the open-boundary pass ride along in the pack kernel?  Needs pass-through
// stores (the kernel then writes inlet / outlet cells anyway) and every outlet
// cell's x-1 neighbour inside the same pack of V cells.
bool can_fuse_open(const mlb_plan *p, int variant)
{
    if (!p->passthrough || variant < 1000 || (p->n_in == 0 && p->n_out == 0))
        return false;
    const int V = pack_cells(p->dtype, variant);
    for (int r = 0; r < 8; r += V)
        if (p->out_xmod8 & (1u << r))
            return false;
    return true;
}

// how far ahead the pack kernels prefetch into L2 (prefetch_ahead), as planes + rows
// (mlb_plan_set_prefetch).  Auto = the cells whose 19 populations make ~10 MB:
// measured on B200 at 512^3 and 256^3 the optimum sits at that many BYTES for
// every storage type (fp32 128 Ki cells, fp64 64 Ki, fp16 192-256 Ki); twice as
// far is already slower than no prefetch (the prefetched lines plus the dirty
// lines of the stores outgrow the L2 share they can hold on to).
void prefetch_distance(const mlb_plan *p, int &dz, int &dy)
{
    const long long cells = p->prefetch >= 0 ? p->prefetch : (512ll << 10) / p->lay.itemsize;
    const long long rows = cells / p->nx;
    dz = (int)(rows / p->ny);
    dy = (int)(rows % p->ny);
}

// pack kernels: one lane per line (0, default) or the bulk form (1; MLB_PF_BULK=1 for
// A/B runs: measured slower at 512^3 for fp32 / fp16 / mixed2 packs)
// Measured on B200 (profiles/pf_bulk_sizes_r2.txt): on SHORT rows the bulk form wins - 128^3 fp32
// two blocks 0.64 -> 0.81 of the HBM peak, 256^3 fp16 storage 0.77 -> 0.81, fp32 storage / fp64
// arithmetic 0.84 -> 0.85 (in place 0.83 -> 0.86) - from 384-cell rows on one lane per line does
// (fp32 256^3 two blocks already prefers it: 0.99 vs 0.975).
int prefetch_bulk(const mlb_plan *p, bool inplace)
{
    static const int v = std::getenv("MLB_PF_BULK") ? std::atoi(std::getenv("MLB_PF_BULK")) : -1;
    if (v >= 0)
        return v;
    if (inplace)
        return p->dtype == MLB_F32C64 && p->nx <= 256;
    if (p->dtype == MLB_F32)
        return p->nx <= 128;
    return p->nx <= 256;
}

template <typename TS>
void fill_args(mlb_plan *p, const void *fpre, void *fpost, int z0, bool fuse_open,
               mlb::StepArgs<TS> &a)
{
    using T = typename mlb::Store<TS>::C;
    for (int q = 0; q < MLB_Q; ++q) {
        a.pre[q] = static_cast<const TS *>(fpre) + (long long)q * p->lay.pop;
        a.post[q] = static_cast<TS *>(fpost) + (long long)q * p->lay.pop;
    }
    a.ct = cls_tab(p);
    a.g = p->g;
    a.z0 = z0;
    a.passthrough = p->passthrough;
    a.fuse_open = fuse_open ? 1 : 0;
    prefetch_distance(p, a.pf_dz, a.pf_dy);
    a.pf_bulk = prefetch_bulk(p, false);
    T cv[MLB_Q];
    inlet_values<T>(p->inlet_u, cv);  // compute dtype, then storage dtype (engine.py:167-171)
    for (int q = 0; q < MLB_Q; ++q)
        a.inlet[q] = mlb::Store<TS>::down(cv[q]);
    a.omega = T(p->omega);
    wall_terms<T>(p->wall_u, a.k);
    a.work = nullptr;
}

// the neighbours' halo planes a launch also stores into (mlb_step_push_range)
struct PushTarget {
    void *below = nullptr, *above = nullptr;  // the neighbours' post blocks (peer memory)
    int nz_below = 0, nz_above = 0;
};

template <typename TS>
void fill_push(const mlb_plan *p, const PushTarget &t, mlb::PushArgs<TS> &ph)
{
    const long long plane = p->lay.plane;
    for (int j = 0; j < 5; ++j) {
        // slab below: its halo plane lz = nz (storage nz_below + 1) takes our plane 0, c_z = -1
        ph.lo[j] = t.below ? static_cast<TS *>(t.below)
                                 + ((long long)mlb::halo_down(j) * (t.nz_below + 2)
                                    + (t.nz_below + 1)) * plane
                           : nullptr;
        // slab above: its halo plane lz = -1 (storage 0) takes our plane nz-1, c_z = +1
        ph.hi[j] = t.above ? static_cast<TS *>(t.above)
                                 + (long long)mlb::halo_up(j) * (t.nz_above + 2) * plane
                           : nullptr;
    }
}

template <typename TS, int V, bool PUSH>
int launch_vec(mlb_plan *p, const mlb::StepArgs<TS> &a, const mlb::PushArgs<TS> &ph, int lx,
               int nplanes, cudaStream_t st)
{
    const int rows = 128 / lx;  // rows per 128-thread block
    // pass-through launches cover the padded row (see step_vec_kernel); a row the
    // pack does not divide ends in a pack of real cells + padding
    const long long cols = a.passthrough ? p->lay.xp : p->nx;
    const dim3 grid((unsigned)(((cols + V - 1) / V + lx - 1) / lx), (p->ny + rows - 1) / rows,
                    nplanes);
    if (lx == 8) mlb::step_vec_kernel<TS, V, 8, PUSH><<<grid, 128, 0, st>>>(a, ph);
    else if (lx == 16) mlb::step_vec_kernel<TS, V, 16, PUSH><<<grid, 128, 0, st>>>(a, ph);
    else mlb::step_vec_kernel<TS, V, 32, PUSH><<<grid, 128, 0, st>>>(a, ph);
    MLB_LAUNCHED();
    return MLB_OK;
}

template <typename TS, bool PUSH>
int launch_scalar(mlb_plan *p, const mlb::StepArgs<TS> &a, const mlb::PushArgs<TS> &ph, int bx,
                  int nplanes, cudaStream_t st)
{
    while (bx > 32 && bx / 2 >= p->nx)
        bx /= 2;
    const long long cols = a.passthrough ? p->lay.xp : p->nx;   // pass-through covers the padded row
    const dim3 grid((unsigned)((cols + bx - 1) / bx), p->ny, nplanes);
    switch (bx) {
    case 32: mlb::step_kernel<TS, 32, PUSH><<<grid, 32, 0, st>>>(a, ph); break;
    case 64: mlb::step_kernel<TS, 64, PUSH><<<grid, 64, 0, st>>>(a, ph); break;
    case 128: mlb::step_kernel<TS, 128, PUSH><<<grid, 128, 0, st>>>(a, ph); break;
    case 256: mlb::step_kernel<TS, 256, PUSH><<<grid, 256, 0, st>>>(a, ph); break;
    default: mlb::step_kernel<TS, 512, PUSH><<<grid, 512, 0, st>>>(a, ph); break;
    }
    MLB_LAUNCHED();
    return MLB_OK;
}

template <typename TS, int V>
int launch_stage(mlb_plan *p, mlb::StepArgs<TS> &a, int nplanes, cudaStream_t st)
{
    using SS = mlb::StageShape<TS, V>;
    static const int group_env = std::getenv("MLB_STAGE_GROUP") ? std::atoi(std::getenv("MLB_STAGE_GROUP")) : 0;
    const int group = group_env > 0 ? group_env : 2;         // warp rows handed out per counter fetch (measured: 2 is best)
    const long long cols = a.passthrough ? p->lay.xp : p->nx;
    const int ncol = (int)((cols + SS::W - 1) / SS::W);
    const long long ntasks = (long long)ncol * p->ny * nplanes;
    if (ntasks >= (1ll << 30))
        return fail(MLB_EUNSUPPORTED, "the staged kernel counts at most 2^30 warp rows per launch");
    const size_t smem = stage_smem<TS, V>();
    auto kernel = mlb::step_stage_kernel<TS, V>;
    if (smem > (48u << 10))
        MLB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // the launch's work counter: one slot of a small ring, so that launches in flight on
    // different streams (boundary planes / interior of a slab) do not share one
    unsigned int *slot = p->d_work + (p->work_next++ & 63);
    MLB_CUDA(cudaMemsetAsync(slot, 0, sizeof(unsigned int), st));
    a.work = slot;
    // as many blocks as can be resident (4 per SM), or fewer for a small launch
    const long long want = (ntasks + 4 * group - 1) / (4 * group);
    const long long blocks = want < 4ll * p->sms ? want : 4ll * p->sms;
    kernel<<<(unsigned)blocks, 128, smem, st>>>(a, group, ncol, (int)ntasks);
    MLB_LAUNCHED();
    return MLB_OK;
}

template <typename TS, int V1, int V2, bool PUSH>
int launch_typed(mlb_plan *p, const void *fpre, void *fpost, int z0, int z1, cudaStream_t st,
                 bool fuse_open, int variant, const PushTarget *push)
{
    mlb::StepArgs<TS> a;
    fill_args<TS>(p, fpre, fpost, z0, fuse_open, a);

    if (variant == VARIANT_STAGED) {
        constexpr int V = sizeof(TS) == 8 || std::is_same<TS, mlb::f32w>::value ? 2 : 4;
        if constexpr (!PUSH && mlb::StageShape<TS, V>::OK) {
            static const int pf = std::getenv("MLB_STAGE_PF") ? std::atoi(std::getenv("MLB_STAGE_PF")) : 0;
            if (!pf) a.pf_dz = a.pf_dy = 0;
            return launch_stage<TS, V>(p, a, z1 - z0, st);
        }
    }
    mlb::PushArgs<TS> ph{};
    if (PUSH)
        fill_push<TS>(p, *push, ph);
    const int lx = variant % 1000, n = z1 - z0;
    if (variant >= 1000) {
        // the pack width the variant means for this dtype: one of the two built
        if (pack_cells(p->dtype, variant) == V1) return launch_vec<TS, V1, PUSH>(p, a, ph, lx, n, st);
        return launch_vec<TS, V2, PUSH>(p, a, ph, lx, n, st);
    }
    // one cell per thread: 19 per-line prefetches per 32 cells cost too many issue
    // slots there, so these kernels use the bulk form - one instruction per
    // population and row (measured at 511^3, fraction of the HBM peak: fp32 0.966
    // without -> 0.982, fp64 1.006 -> 1.014, fp32 storage / fp64 arithmetic 0.837
    // -> 0.888) - except with fp16 storage, where any prefetch loses (0.62 -> 0.57)
    a.pf_bulk = 1;
    if (sizeof(TS) == 2)
        a.pf_dz = a.pf_dy = 0;
    return launch_scalar<TS, PUSH>(p, a, ph, variant, n, st);
}

int launch_step(mlb_plan *p, const void *fpre, void *fpost, int z0, int z1, cudaStream_t st,
                bool fuse_open = false, const PushTarget *push = nullptr)
{
    // (a launch that also pushes into the neighbours' halos keeps the direct kernel)
    const int variant = resolve_variant(p, push == nullptr);
    if (!variant_exists(p->dtype, variant))
        return fail(MLB_EINVAL, "kernel variant %d does not exist for dtype code %d", variant,
                    p->dtype);
    // pack widths per dtype: W = 1 -> 16-byte packs (fp32 / fp64); fp16 storage
    // has W = 2 (4 halves) and W = 3 (2 halves)
    if (p->dtype == MLB_F32)
        return push ? launch_typed<float, 4, 2, true>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push)
                    : launch_typed<float, 4, 2, false>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push);
    if (p->dtype == MLB_F64)
        return push ? launch_typed<double, 2, 2, true>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push)
                    : launch_typed<double, 2, 2, false>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push);
    if (p->dtype == MLB_F32C64)
        return push ? launch_typed<mlb::f32w, 2, 2, true>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push)
                    : launch_typed<mlb::f32w, 2, 2, false>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push);
    return push ? launch_typed<__half, 4, 2, true>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push)
                : launch_typed<__half, 4, 2, false>(p, fpre, fpost, z0, z1, st, fuse_open, variant, push);
}

// in-place (AA pattern) launches: kind 0 = R0 -> R1 step, 1 = R1 -> R0 step, 2 = swap
// plane range and ring neighbours of one in-place launch (z-slabs; all-zero =
// the whole domain on one GPU)
struct AaRange {
    int z0 = 0, z1 = -1;                      // z1 < 0: all planes
    void *below = nullptr, *above = nullptr;  // the neighbours' blocks (peer memory)
    int nz_below = 0, nz_above = 0;
};

template <typename TS>
void fill_aa(mlb_plan *p, void *f, const AaRange &r, mlb::AAArgs<TS> &a)
{
    using T = typename mlb::Store<TS>::C;
    for (int q = 0; q < MLB_Q; ++q)
        a.f[q] = static_cast<TS *>(f) + (long long)q * p->lay.pop;
    a.ct = cls_tab(p);
    a.g = p->g;
    a.omega = T(p->omega);
    wall_terms<T>(p->wall_u, a.k);
    T cv[MLB_Q];
    inlet_values<T>(p->inlet_u, cv);  // compute dtype, then storage dtype (engine.py:167-171)
    for (int q = 0; q < MLB_Q; ++q)
        a.inlet[q] = mlb::Store<TS>::down(cv[q]);
    a.z0 = r.z0;
    prefetch_distance(p, a.pf_dz, a.pf_dy);
    a.pf_bulk = prefetch_bulk(p, true);
    const long long plane = p->lay.plane;
    for (int j = 0; j < 5; ++j) {
        // slab below: its top plane lz = nz_below-1 (storage nz_below), c_z = +1 populations
        a.lo[j] = r.below ? static_cast<TS *>(r.below)
                                + ((long long)mlb::halo_up(j) * (r.nz_below + 2) + r.nz_below) * plane
                          : nullptr;
        // slab above: its bottom plane lz = 0 (storage 1), c_z = -1 populations
        a.hi[j] = r.above ? static_cast<TS *>(r.above)
                                + ((long long)mlb::halo_down(j) * (r.nz_above + 2) + 1) * plane
                          : nullptr;
    }
}

template <typename TS>
int launch_aa(mlb_plan *p, void *f, int kind, const AaRange &r, cudaStream_t st)
{
    mlb::AAArgs<TS> a;
    fill_aa<TS>(p, f, r, a);
    constexpr int BX = 128;
    const int n = (r.z1 < 0 ? p->nz : r.z1) - r.z0;
    const dim3 grid((p->nx + BX - 1) / BX, p->ny, n);
    const bool remote = r.below || r.above;
    if (kind == 0) mlb::aa_pull_kernel<TS, BX><<<grid, BX, 0, st>>>(a);
    else if (kind == 1) mlb::aa_local_kernel<TS, BX><<<grid, BX, 0, st>>>(a);
    else if (remote) mlb::aa_swap_kernel<TS, BX, true><<<grid, BX, 0, st>>>(a);
    else mlb::aa_swap_kernel<TS, BX, false><<<grid, BX, 0, st>>>(a);
    MLB_LAUNCHED();
    return MLB_OK;
}

// layout of the in-place pull half: row blocks (mlb_plan_set_inplace_layout; MLB_AA_ROWB
// overrides for A/B runs)
bool aa_row_blocks(const mlb_plan *p)
{
    static const int env = std::getenv("MLB_AA_ROWB") ? std::atoi(std::getenv("MLB_AA_ROWB")) : -1;
    const int mode = env >= 0 ? env : p->aa_layout;
    return mode == 1;
}

template <typename TS, int V, int LX>
int launch_aa_vec(mlb_plan *p, void *f, int kind, const AaRange &r, cudaStream_t st)
{
    mlb::AAArgs<TS> a;
    fill_aa<TS>(p, f, r, a);
    const int rows = 128 / LX;
    const int n = (r.z1 < 0 ? p->nz : r.z1) - r.z0;
    // the local half covers the padded row (it rewrites the padding: whole last lines)
    const long long cols = kind == 1 ? p->lay.xp : p->nx;
    const dim3 grid((unsigned)(((cols + V - 1) / V + LX - 1) / LX), (p->ny + rows - 1) / rows, n);
    const bool remote = r.below || r.above;
    if (kind == 0 && aa_row_blocks(p)) {
        // pull half, row-block layout: a block is WPR warps side by side in x (values that
        // cross a warp boundary go through shared memory) times 4 / WPR rows
        const int ppr = (p->nx + V - 1) / V;
        const int wpr = ppr <= 32 ? 1 : ppr <= 64 ? 2 : 4;
        const dim3 rgrid((ppr + 32 * wpr - 1) / (32 * wpr), (p->ny + 4 / wpr - 1) / (4 / wpr), n);
#define MLB_ROWB(W)                                                                      \
        if (remote) mlb::aa_pull_vec_kernel<TS, V, 32, true, W><<<rgrid, 128, 0, st>>>(a); \
        else mlb::aa_pull_vec_kernel<TS, V, 32, false, W><<<rgrid, 128, 0, st>>>(a);
        if (wpr == 1) { MLB_ROWB(1) } else if (wpr == 2) { MLB_ROWB(2) } else { MLB_ROWB(4) }
#undef MLB_ROWB
    } else if (kind == 0) {
        // pull half: results for crossing directions go into the neighbours' planes
        if (remote) mlb::aa_pull_vec_kernel<TS, V, LX, true><<<grid, 128, 0, st>>>(a);
        else mlb::aa_pull_vec_kernel<TS, V, LX, false><<<grid, 128, 0, st>>>(a);
    } else {
        // local half: back in the normal representation; boundary planes also fill
        // the neighbours' halo planes (the two-buffer kernel's push)
        mlb::PushArgs<TS> ph{};
        if (remote) {
            PushTarget t;
            if (r.z0 == 0) { t.below = r.below; t.nz_below = r.nz_below; }
            if ((r.z1 < 0 ? p->nz : r.z1) == p->nz) { t.above = r.above; t.nz_above = r.nz_above; }
            fill_push<TS>(p, t, ph);
            mlb::aa_local_vec_kernel<TS, V, LX, true><<<grid, 128, 0, st>>>(a, ph);
        } else {
            mlb::aa_local_vec_kernel<TS, V, LX, false><<<grid, 128, 0, st>>>(a, ph);
        }
    }
    MLB_LAUNCHED();
    return MLB_OK;
}

template <typename TS, int V>
int launch_aa_vec_lx(mlb_plan *p, void *f, int kind, int lx, const AaRange &r, cudaStream_t st)
{
    if (lx == 8) return launch_aa_vec<TS, V, 8>(p, f, kind, r, st);
    if (lx == 16) return launch_aa_vec<TS, V, 16>(p, f, kind, r, st);
    return launch_aa_vec<TS, V, 32>(p, f, kind, r, st);
}

// the variant the in-place kernels run with (0 = auto: packs whenever the row
// length allows)
int resolve_aa_variant(const mlb_plan *p)
{
    if (p->variant != 0 && p->variant != VARIANT_STAGED)
        return p->variant;
    // packs for any row length (a ragged row ends in a pack of real cells + padding)
    if (p->nx >= 128) return p->dtype == MLB_F32 || p->dtype == MLB_F64 ? 1016 : 2016;
    return 128;
}

bool aa_uses_packs(const mlb_plan *p, int variant)
{
    return variant >= 1000 && variant_exists(p->dtype, variant)
        && p->nx >= pack_cells(p->dtype, variant);
}

// Open boundaries in place: the pack kernels apply the pass inside the step
// (inlet cells take the constant, outlet cells copy their x-1 neighbour inside
// the pack), which needs every outlet cell's x-1 neighbour in the same pack and
// no outlet cell copying from another outlet cell.
bool aa_open_ok(const mlb_plan *p, int variant)
{
    if (p->n_in == 0 && p->n_out == 0)
        return true;
    if (!aa_uses_packs(p, variant) || p->out_chained)
        return false;
    const int V = pack_cells(p->dtype, variant);
    for (int r = 0; r < 8; r += V)
        if (p->out_xmod8 & (1u << r))
            return false;
    return true;
}

// the in-place step kernels follow the plan's variant: pack kernels when the
// two-buffer path would use one (the swap is always scalar)
int launch_aa_any(mlb_plan *p, void *f, int kind, cudaStream_t st, const AaRange &r = AaRange())
{
    const int variant = resolve_aa_variant(p);
    if (!variant_exists(p->dtype, variant))
        return fail(MLB_EINVAL, "kernel variant %d does not exist for dtype code %d", variant,
                    p->dtype);
    const bool vec = kind != 2 && aa_uses_packs(p, variant);
    const int lx = variant % 1000;
    if (p->dtype == MLB_F32) {
        if (vec && pack_cells(p->dtype, variant) == 2)
            return launch_aa_vec_lx<float, 2>(p, f, kind, lx, r, st);
        return vec ? launch_aa_vec_lx<float, 4>(p, f, kind, lx, r, st)
                   : launch_aa<float>(p, f, kind, r, st);
    }
    if (p->dtype == MLB_F64)
        return vec ? launch_aa_vec_lx<double, 2>(p, f, kind, lx, r, st)
                   : launch_aa<double>(p, f, kind, r, st);
    if (p->dtype == MLB_F32C64)
        return vec ? launch_aa_vec_lx<mlb::f32w, 2>(p, f, kind, lx, r, st)
                   : launch_aa<mlb::f32w>(p, f, kind, r, st);
    if (vec && variant >= 3000) return launch_aa_vec_lx<__half, 2>(p, f, kind, lx, r, st);
    if (vec) return launch_aa_vec_lx<__half, 4>(p, f, kind, lx, r, st);
    return launch_aa<__half>(p, f, kind, r, st);
}

template <typename T>
int launch_open(mlb_plan *p, void *fpost, int z0, int z1, cudaStream_t st)
{
    using C = typename mlb::Store<T>::C;
    T *f = static_cast<T *>(fpost);
    const long long i0 = p->in_zoff[z0], i1 = p->in_zoff[z1];
    if (i1 > i0) {
        // computed in compute dtype, stored in storage dtype (engine.py:167-171)
        C cv[MLB_Q];
        inlet_values<C>(p->inlet_u, cv);
        mlb::InletVals<T> v;
        for (int q = 0; q < MLB_Q; ++q)
            v.v[q] = mlb::Store<T>::down(cv[q]);
        const long long n = i1 - i0;
        mlb::inlet_kernel<T><<<(unsigned)((n + 127) / 128), 128, 0, st>>>(
            f, p->d_in + i0, n, p->lay.pop, v);
        MLB_LAUNCHED();
    }
    const long long o0 = p->out_zoff[z0], o1 = p->out_zoff[z1];
    if (o1 > o0) {
        const long long n = o1 - o0;
        const unsigned blocks = (unsigned)((n + 127) / 128);
        // (each plane range its own part of the scratch: the boundary planes and the
        // interior of a slab run this pass concurrently on two streams)
        T *tmp = p->d_out_tmp ? static_cast<T *>(p->d_out_tmp) + o0 : nullptr;
        if (!p->out_chained) {
            mlb::outlet_kernel<T><<<blocks, 128, 0, st>>>(f, tmp, p->d_out + o0, n,
                                                          p->lay.pop, p->n_out, 0);
            MLB_LAUNCHED();
        } else {
            mlb::outlet_kernel<T><<<blocks, 128, 0, st>>>(f, tmp, p->d_out + o0, n,
                                                          p->lay.pop, p->n_out, 1);
            MLB_LAUNCHED();
            mlb::outlet_kernel<T><<<blocks, 128, 0, st>>>(f, tmp, p->d_out + o0, n,
                                                          p->lay.pop, p->n_out, 2);
            MLB_LAUNCHED();
        }
    }
    return MLB_OK;
}

int check_plan(const mlb_plan *p, bool need_flags)
{
    if (!p)
        return fail(MLB_EINVAL, "plan is NULL");
    if (need_flags && !p->have_flags)
        return fail(MLB_EINVAL, "plan has no flags: call mlb_plan_set_flags first");
    return MLB_OK;
}

int copy_dense(const mlb_plan *p, const void *src, void *dst, bool to_device,
               cudaStream_t st)
{
    const int sz = p->lay.itemsize;
    const size_t row = (size_t)p->nx * sz;
    const size_t rows = (size_t)p->nz * p->ny;
    const size_t dense_pop = rows * row;
    for (int q = 0; q < MLB_Q; ++q) {
        const char *h = static_cast<const char *>(to_device ? src : dst) + q * dense_pop;
        const char *d = static_cast<const char *>(to_device ? dst : src)
                      + ((size_t)q * p->lay.pop + p->lay.plane) * sz;
        if (p->lay.xp == p->nx) {
            if (to_device)
                MLB_CUDA(cudaMemcpyAsync((void *)d, h, dense_pop, cudaMemcpyHostToDevice, st));
            else
                MLB_CUDA(cudaMemcpyAsync((void *)h, d, dense_pop, cudaMemcpyDeviceToHost, st));
        } else {
            if (to_device)
                MLB_CUDA(cudaMemcpy2DAsync((void *)d, (size_t)p->lay.xp * sz, h, row, row, rows,
                                           cudaMemcpyHostToDevice, st));
            else
                MLB_CUDA(cudaMemcpy2DAsync((void *)h, row, d, (size_t)p->lay.xp * sz, row, rows,
                                           cudaMemcpyDeviceToHost, st));
        }
    }
    return MLB_OK;
}

}  // namespace

extern "C" {

const char *mlb_last_error(void) { return g_err; }
int mlb_abi_version(void) { return MLB_ABI_VERSION; }
#ifndef MLB_BUILD_ID
#define MLB_BUILD_ID "unknown"
#endif
const char *mlb_build_id(void) { return MLB_BUILD_ID; }
int64_t mlb_launch_count(void) { return g_launches.load(); }

int mlb_layout_query(int nx, int ny, int nz, int dtype, mlb_layout *out)
{
    if (!out)
        return fail(MLB_EINVAL, "out is NULL");
    return layout_of(nx, ny, nz, dtype, out);
}

int mlb_plan_create(mlb_plan **out, int nx, int ny, int nz, int dtype, double omega,
                    const double wall_u[3], double inlet_u, int device, int z_mode)
{
    if (!out)
        return fail(MLB_EINVAL, "out is NULL");
    *out = nullptr;
    if (z_mode != MLB_Z_PERIODIC && z_mode != MLB_Z_HALO)
        return fail(MLB_EINVAL, "unknown z_mode %d", z_mode);
    mlb_layout lay;
    if (int rc = layout_of(nx, ny, nz, dtype, &lay))
        return rc;
    int ndev = 0;
    MLB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(MLB_EINVAL, "device %d out of range (%d visible)", device, ndev);
    MLB_ON_DEVICE(device);
    mlb_plan *p = new (std::nothrow) mlb_plan;
    if (!p)
        return fail(MLB_ENOMEM, "out of host memory");
    p->nx = nx; p->ny = ny; p->nz = nz; p->dtype = dtype;
    p->device = device; p->z_mode = z_mode; p->lay = lay;
    set_geom(p);
    if (int rc = mlb_plan_set_physics(p, omega, wall_u, inlet_u)) {
        delete p;
        return rc;
    }
    cudaDeviceGetAttribute(&p->sms, cudaDevAttrMultiProcessorCount, device);
    p->diag_blocks = p->sms * 8;
    cudaError_t e = pool_alloc(&p->d_partials, sizeof(double) * mlb::DIAG_N * p->diag_blocks);
    if (e == cudaSuccess) e = pool_alloc(&p->d_diag, sizeof(double) * mlb::DIAG_N);
    if (e == cudaSuccess) e = pool_alloc(&p->d_work, 64 * sizeof(unsigned int));
    if (e == cudaSuccess) e = cudaEventCreate(&p->ev0);
    if (e == cudaSuccess) e = cudaEventCreate(&p->ev1);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        mlb_plan_destroy(p);
        return fail(MLB_ECUDA, "plan setup: %s", cudaGetErrorString(e));
    }
    *out = p;
    return MLB_OK;
}

int mlb_plan_destroy(mlb_plan *p)
{
    if (!p)
        return MLB_OK;
    DeviceGuard guard_(p->device);
    // cudaFree used to wait for work still using the tables; a pooled block can be
    // handed to the next plan at once, so wait here
    cudaDeviceSynchronize();
    pool_free(p->d_flags); pool_free(p->d_cls); pool_free(p->d_mlinks); pool_free(p->d_in);
    pool_free(p->d_kind); pool_free(p->d_tab);
    pool_free(p->d_out); pool_free(p->d_out_tmp); pool_free(p->d_partials); pool_free(p->d_diag);
    pool_free(p->d_work);
    if (p->ev0) cudaEventDestroy(p->ev0);
    if (p->ev1) cudaEventDestroy(p->ev1);
    if (p->ev_fork) cudaEventDestroy(p->ev_fork);
    if (p->ev_join) cudaEventDestroy(p->ev_join);
    if (p->gc.exec) cudaGraphExecDestroy(p->gc.exec);
    if (p->cap_stream) cudaStreamDestroy(p->cap_stream);
    if (p->up_stream) cudaStreamDestroy(p->up_stream);
    if (p->down_stream) cudaStreamDestroy(p->down_stream);
    delete p;
    return MLB_OK;
}

int mlb_plan_get_layout(const mlb_plan *p, mlb_layout *out)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!out) return fail(MLB_EINVAL, "out is NULL");
    *out = p->lay;
    return MLB_OK;
}

int mlb_plan_set_physics(mlb_plan *p, double omega, const double wall_u[3], double inlet_u)
{
    if (int rc = check_plan(p, false)) return rc;
    // omega = 0 is legal kernel input (pure streaming, test_kernels.py:152-164)
    if (!(omega >= 0.0 && omega < 2.0))
        return fail(MLB_EINVAL, "relaxation rate omega=%g outside [0, 2)", omega);
    ++p->epoch;
    p->omega = omega;
    for (int i = 0; i < 3; ++i)
        p->wall_u[i] = wall_u ? wall_u[i] : 0.0;
    p->inlet_u = inlet_u;
    return MLB_OK;
}

int mlb_plan_set_variant(mlb_plan *p, int variant)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!variant_exists(p->dtype, variant))
        return fail(MLB_EINVAL, "variant %d: must be 0 (auto), a block width in {32,64,128,256,"
                    "512} (one cell per thread), or W*1000 + {8,16,32} with W = 1 (16-byte packs, "
                    "fp32/fp64), 2 or 3 (8- / 4-byte packs, fp16 storage)", variant);
    p->variant = variant;
    ++p->epoch;
    return MLB_OK;
}

const char *mlb_plan_kernel_name(const mlb_plan *p)
{
    static thread_local char name[64];
    if (!p) return "";
    const int v = resolve_variant(p);
    const char *t = p->dtype == MLB_F32 ? "float" : p->dtype == MLB_F64 ? "double"
                  : p->dtype == MLB_F32C64 ? "f32w" : "__half";
    if (v == VARIANT_STAGED)
        snprintf(name, sizeof(name), "mlb::step_stage_kernel<%s, %d>", t, pack_cells(p->dtype, v));
    else if (v >= 1000)
        snprintf(name, sizeof(name), "mlb::step_vec_kernel<%s, %d, %d, false>", t,
                 pack_cells(p->dtype, v), v % 1000);
    else
        snprintf(name, sizeof(name), "mlb::step_kernel<%s, %d, false>", t, v);
    return name;
}

int mlb_plan_set_passthrough(mlb_plan *p, int on)
{
    if (int rc = check_plan(p, false)) return rc;
    if (on && p->out_chained)
        return fail(MLB_EUNSUPPORTED, "pass-through stores are not valid for this geometry: an "
                    "outlet cell copies from another outlet cell, and the reference then reads "
                    "that cell's STALE value in fpost (numpy evaluates the right-hand side "
                    "first, engine.py:179-180), which pass-through would refresh");
    p->passthrough = on ? 1 : 0;
    ++p->epoch;
    return MLB_OK;
}

int mlb_plan_set_prefetch(mlb_plan *p, long long cells)
{
    if (int rc = check_plan(p, false)) return rc;
    if (cells < -1)
        return fail(MLB_EINVAL, "prefetch distance %lld: must be -1 (auto), 0 (off) or a number "
                    "of cells", cells);
    p->prefetch = cells;
    ++p->epoch;
    return MLB_OK;
}

int mlb_plan_set_flags(mlb_plan *p, const uint8_t *h_flags, const uint8_t *h_lo,
                       const uint8_t *h_hi)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!h_flags)
        return fail(MLB_EINVAL, "h_flags is NULL");
    MLB_ON_DEVICE(p->device);
    const int nx = p->nx, ny = p->ny, nz = p->nz;
    const long long xp = p->lay.xp, plane = p->lay.plane;
    const size_t padded = (size_t)(nz + 2) * plane;
    const size_t dense_plane = (size_t)nx * ny;
    const uint8_t *src_lo = h_lo ? h_lo : h_flags + (size_t)(nz - 1) * dense_plane;
    const uint8_t *src_hi = h_hi ? h_hi : h_flags;

    if (p->have_flags)
        MLB_CUDA(cudaDeviceSynchronize());   // earlier launches may still read the old tables
    pool_free(p->d_flags); pool_free(p->d_cls); pool_free(p->d_mlinks); pool_free(p->d_in);
    pool_free(p->d_kind); pool_free(p->d_tab);
    pool_free(p->d_out); pool_free(p->d_out_tmp);
    p->d_flags = nullptr; p->d_cls = p->d_mlinks = nullptr; p->d_in = p->d_out = nullptr;
    p->d_kind = nullptr; p->d_tab = nullptr;
    p->d_out_tmp = nullptr;
    p->have_flags = false;
    p->n_in = p->n_out = 0;
    ++p->epoch;

    // the padded flag block on the device, straight from the caller's dense
    // array (row padding = solid, never written); no padded host copy
    MLB_CUDA(pool_alloc(&p->d_flags, padded));
    if (xp != nx)
        MLB_CUDA(cudaMemset(p->d_flags, 1, padded));
    if (xp == nx)
        MLB_CUDA(cudaMemcpy(p->d_flags + plane, h_flags, (size_t)nz * dense_plane,
                            cudaMemcpyHostToDevice));
    else
        MLB_CUDA(cudaMemcpy2D(p->d_flags + plane, (size_t)xp, h_flags, (size_t)nx, (size_t)nx,
                              (size_t)nz * ny, cudaMemcpyHostToDevice));
    MLB_CUDA(cudaMemcpy2D(p->d_flags, (size_t)xp, src_lo, (size_t)nx, (size_t)nx, (size_t)ny,
                          cudaMemcpyHostToDevice));
    MLB_CUDA(cudaMemcpy2D(p->d_flags + (size_t)(nz + 1) * plane, (size_t)xp, src_hi, (size_t)nx,
                          (size_t)nx, (size_t)ny, cudaMemcpyHostToDevice));

    // census on the device: open-boundary cells (inlet / outlet index lists are
    // needed only if there are any) and invalid codes.  A cavity or a periodic
    // box never walks its flags on the host.
    unsigned long long *d_census = nullptr, census[3] = {0, 0, 0};
    MLB_CUDA(pool_alloc(&d_census, sizeof(census)));
    MLB_CUDA(cudaMemset(d_census, 0, sizeof(census)));
    {
        const dim3 cgrid((unsigned)((xp + 255) / 256), ny, nz + 2);
        mlb::flag_census_kernel<<<cgrid, 256>>>(p->d_flags, p->g, d_census);
        MLB_LAUNCHED();
    }
    MLB_CUDA(cudaMemcpy(census, d_census, sizeof(census), cudaMemcpyDeviceToHost));
    pool_free(d_census);

    {
        auto wall_plane = [&](const uint8_t *pl) {
            for (size_t i = 0; i < dense_plane; ++i)
                if (pl[i] != 1 && pl[i] != 2) return false;
            return true;
        };
        p->z_closed = p->z_mode == MLB_Z_PERIODIC && nz >= 2 && wall_plane(h_flags)
                      && wall_plane(h_flags + (size_t)(nz - 1) * dense_plane);
    }
    std::vector<long long> in_idx, out_idx;
    p->in_zoff.assign(nz + 1, 0);
    p->out_zoff.assign(nz + 1, 0);
    p->out_xmod8 = 0;
    if (census[0] || census[1] || census[2]) {
        in_idx.reserve(census[0]);
        out_idx.reserve(census[1]);
        for (int sz = 0; sz < nz + 2; ++sz) {
            const uint8_t *src = sz == 0 ? src_lo : sz == nz + 1 ? src_hi
                                                  : h_flags + (size_t)(sz - 1) * dense_plane;
            const bool interior = sz >= 1 && sz <= nz;
            if (interior) {
                p->in_zoff[sz - 1] = (long long)in_idx.size();
                p->out_zoff[sz - 1] = (long long)out_idx.size();
            }
            for (int y = 0; y < ny; ++y) {
                const uint8_t *row = src + (size_t)y * nx;
                const long long d0 = (long long)sz * plane + (long long)y * xp;
                // rows of plain fluid / solid / lid cells (all but a few) need no
                // per-cell work: one vectorisable scan finds the exceptions
                uint8_t special = 0;
                for (int x = 0; x < nx; ++x)
                    special |= (uint8_t)(row[x] >= 3);
                if (!special)
                    continue;
                for (int x = 0; x < nx; ++x) {
                    const uint8_t m = row[x];
                    if (m > 4)
                        return fail(MLB_EINVAL, "flag array holds unknown cell code %d at "
                                    "(x=%d, y=%d, plane=%d)", (int)m, x, y, sz - 1);
                    if (!interior)
                        continue;
                    if (m == 3)
                        in_idx.push_back(d0 + x);
                    else if (m == 4) {
                        p->out_xmod8 |= 1u << (x & 7);
                        if (x == 0)
                            return fail(MLB_EUNSUPPORTED, "outlet cell at x = 0 (y=%d, z=%d): "
                                        "its source would be the previous row's last cell", y,
                                        sz - 1);
                        out_idx.push_back(d0 + x);
                    }
                }
            }
        }
    }
    p->in_zoff[nz] = (long long)in_idx.size();
    p->out_zoff[nz] = (long long)out_idx.size();
    // an outlet cell whose source is itself an outlet cell forces the
    // gather-then-scatter form (numpy evaluates the right-hand side first)
    p->out_chained = false;
    for (size_t j = 1; j < out_idx.size(); ++j)
        if (out_idx[j] - 1 == out_idx[j - 1]) {
            p->out_chained = true;
            break;
        }
    if (p->out_chained)
        p->passthrough = 0;  // see mlb_plan_set_passthrough

    p->n_in = (long long)in_idx.size();
    p->n_out = (long long)out_idx.size();
    if (p->n_in) {
        MLB_CUDA(pool_alloc(&p->d_in, sizeof(long long) * p->n_in));
        MLB_CUDA(cudaMemcpy(p->d_in, in_idx.data(), sizeof(long long) * p->n_in,
                            cudaMemcpyHostToDevice));
    }
    if (p->n_out) {
        MLB_CUDA(pool_alloc(&p->d_out, sizeof(long long) * p->n_out));
        MLB_CUDA(cudaMemcpy(p->d_out, out_idx.data(), sizeof(long long) * p->n_out,
                            cudaMemcpyHostToDevice));
        if (p->out_chained)
            MLB_CUDA(pool_alloc(&p->d_out_tmp, (size_t)p->lay.itemsize * MLB_Q * p->n_out));
    }
    // flags -> one kind byte per cell + the dictionary of distinct (class word,
    // link bits) pairs, in one pass (the class words live in registers)
    const dim3 grid((unsigned)((xp + 127) / 128), ny, nz + 2);
    unsigned int *d_esc = nullptr;
    MLB_CUDA(pool_alloc(&p->d_kind, padded));
    MLB_CUDA(pool_alloc(&p->d_tab, 256 * sizeof(unsigned long long)));
    MLB_CUDA(pool_alloc(&d_esc, sizeof(unsigned int)));
    MLB_CUDA(cudaMemset(p->d_tab, 0xff, 256 * sizeof(unsigned long long)));
    MLB_CUDA(cudaMemset(p->d_tab, 0, sizeof(unsigned long long)));  // slot 0 = bulk (0, 0)
    MLB_CUDA(cudaMemset(d_esc, 0, sizeof(unsigned int)));
    mlb::build_kind_kernel<<<grid, 128>>>(p->d_flags, p->g, p->d_tab, p->d_kind, d_esc, nullptr,
                                          nullptr);
    MLB_LAUNCHED();
    MLB_CUDA(cudaMemcpy(&p->n_escape, d_esc, sizeof(unsigned int), cudaMemcpyDeviceToHost));
    if (p->n_escape) {
        // more than 254 distinct pairs: the overflow cells read full-width words.
        // The table is full now, so a second pass finds the same slots.
        MLB_CUDA(pool_alloc(&p->d_cls, padded * sizeof(uint32_t)));
        MLB_CUDA(pool_alloc(&p->d_mlinks, padded * sizeof(uint32_t)));
        MLB_CUDA(cudaMemset(d_esc, 0, sizeof(unsigned int)));
        mlb::build_kind_kernel<<<grid, 128>>>(p->d_flags, p->g, p->d_tab, p->d_kind, d_esc,
                                              p->d_cls, p->d_mlinks);
        MLB_LAUNCHED();
        MLB_CUDA(cudaMemcpy(&p->n_escape, d_esc, sizeof(unsigned int), cudaMemcpyDeviceToHost));
    }
    pool_free(d_esc);
    unsigned long long tab[256];
    MLB_CUDA(cudaMemcpy(tab, p->d_tab, sizeof(tab), cudaMemcpyDeviceToHost));
    p->n_kinds = 0;
    for (int k = 0; k < 255; ++k)
        p->n_kinds += tab[k] != mlb::KIND_EMPTY;
    pool_free(p->d_flags);  // only the build reads the raw flag block
    p->d_flags = nullptr;
    p->have_flags = true;
    return MLB_OK;
}

int mlb_plan_get_flags(const mlb_plan *p, uint8_t *h_flags)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!h_flags) return fail(MLB_EINVAL, "h_flags is NULL");
    MLB_ON_DEVICE(p->device);
    // from what the kernels read - kind byte -> dictionary (or the full-width
    // word for escape cells) -> low bits: proves the codes the kernel tests
    const size_t padded = (size_t)(p->nz + 2) * p->lay.plane;
    std::vector<uint8_t> kind(padded);
    MLB_CUDA(cudaMemcpy(kind.data(), p->d_kind, padded, cudaMemcpyDeviceToHost));
    unsigned long long tab[256];
    MLB_CUDA(cudaMemcpy(tab, p->d_tab, sizeof(tab), cudaMemcpyDeviceToHost));
    std::vector<uint32_t> full;
    if (p->n_escape) {
        full.resize(padded);
        MLB_CUDA(cudaMemcpy(full.data(), p->d_cls, padded * sizeof(uint32_t),
                            cudaMemcpyDeviceToHost));
    }
    for (int z = 0; z < p->nz; ++z)
        for (int y = 0; y < p->ny; ++y)
            for (int x = 0; x < p->nx; ++x) {
                const size_t d = (size_t)(z + 1) * p->lay.plane + (size_t)y * p->lay.xp + x;
                const uint32_t c = kind[d] == mlb::KIND_ESCAPE ? full[d]
                                                               : (uint32_t)tab[kind[d]];
                h_flags[((size_t)z * p->ny + y) * p->nx + x] = (uint8_t)(c & mlb::CLS_FLAG);
            }
    return MLB_OK;
}

int mlb_plan_geometry_stats(const mlb_plan *p, int64_t out[2])
{
    if (int rc = check_plan(p, true)) return rc;
    if (!out) return fail(MLB_EINVAL, "out is NULL");
    out[0] = p->n_kinds;
    out[1] = p->n_escape;
    return MLB_OK;
}

int mlb_upload(const mlb_plan *p, const void *h_dense, void *d_f, void *stream)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!h_dense || !d_f) return fail(MLB_EINVAL, "NULL buffer");
    MLB_ON_DEVICE(p->device);
    return copy_dense(p, h_dense, d_f, true, S(stream));
}

int mlb_download(const mlb_plan *p, const void *d_f, void *h_dense, void *stream)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!h_dense || !d_f) return fail(MLB_EINVAL, "NULL buffer");
    MLB_ON_DEVICE(p->device);
    return copy_dense(p, d_f, h_dense, false, S(stream));
}

int mlb_step_range(mlb_plan *p, const void *d_fpre, void *d_fpost, int z0, int z1,
                   void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_fpre || !d_fpost) return fail(MLB_EINVAL, "NULL population block");
    if (d_fpre == d_fpost)
        return fail(MLB_EINVAL, "fpre and fpost must be distinct blocks");
    if (z0 < 0 || z1 > p->nz || z0 > z1)
        return fail(MLB_EINVAL, "plane range [%d, %d) outside [0, %d)", z0, z1, p->nz);
    if (z0 == z1) return MLB_OK;
    MLB_ON_DEVICE(p->device);
    return launch_step(p, d_fpre, d_fpost, z0, z1, S(stream));
}

int mlb_step(mlb_plan *p, const void *d_fpre, void *d_fpost, void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    return mlb_step_range(p, d_fpre, d_fpost, 0, p->nz, stream);
}

int mlb_open_pass_range(mlb_plan *p, void *d_fpost, int z0, int z1, void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_fpost) return fail(MLB_EINVAL, "NULL population block");
    if (z0 < 0 || z1 > p->nz || z0 > z1)
        return fail(MLB_EINVAL, "plane range [%d, %d) outside [0, %d)", z0, z1, p->nz);
    if (p->n_in == 0 && p->n_out == 0) return MLB_OK;
    MLB_ON_DEVICE(p->device);
    if (p->dtype == MLB_F32) return launch_open<float>(p, d_fpost, z0, z1, S(stream));
    if (p->dtype == MLB_F64) return launch_open<double>(p, d_fpost, z0, z1, S(stream));
    if (p->dtype == MLB_F32C64) return launch_open<mlb::f32w>(p, d_fpost, z0, z1, S(stream));
    return launch_open<__half>(p, d_fpost, z0, z1, S(stream));
}

int mlb_step_open_range(mlb_plan *p, const void *d_fpre, void *d_fpost, int z0, int z1,
                        void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (can_fuse_open(p, resolve_variant(p))) {
        if (!d_fpre || !d_fpost) return fail(MLB_EINVAL, "NULL population block");
        if (d_fpre == d_fpost)
            return fail(MLB_EINVAL, "fpre and fpost must be distinct blocks");
        if (z0 < 0 || z1 > p->nz || z0 > z1)
            return fail(MLB_EINVAL, "plane range [%d, %d) outside [0, %d)", z0, z1, p->nz);
        if (z0 == z1) return MLB_OK;
        MLB_ON_DEVICE(p->device);
        return launch_step(p, d_fpre, d_fpost, z0, z1, S(stream), true);
    }
    if (int rc = mlb_step_range(p, d_fpre, d_fpost, z0, z1, stream)) return rc;
    return mlb_open_pass_range(p, d_fpost, z0, z1, stream);
}

int mlb_open_pass(mlb_plan *p, void *d_fpost, void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    return mlb_open_pass_range(p, d_fpost, 0, p->nz, stream);
}

// ---- CUDA graphs for launch-bound domains ------------------------------------
// Below a few million cells a step takes tens of microseconds or less and the
// loop is bound by launch latency, not by HBM (the reference's loop has the same
// problem with Python overhead, engine.py:244-249 / SURVEY "timing semantics").
// mlb_run_steps / mlb_run_steps_inplace then capture a run of steps - the very
// launches the plain loop makes: same kernels, same arguments, same order, so
// the same bits - into a CUDA graph once, and replay it.
namespace {

constexpr int GRAPH_STEPS = 32;                  // steps per replayed graph
constexpr long long GRAPH_AUTO_CELLS = 4ll << 20;  // auto: domains up to this many cells

int one_step(mlb_plan *p, void *pre, void *post, void *stream)
{
    return mlb_step_open_range(p, pre, post, 0, p->nz, stream);
}

bool graph_wanted(const mlb_plan *p, int nsteps)
{
    static const int env = std::getenv("MLB_GRAPH") ? std::atoi(std::getenv("MLB_GRAPH")) : -1;
    const int mode = env >= 0 ? env : p->graph_mode;
    if (mode == 0 || nsteps < 8)
        return false;
    return mode == 1 || (long long)p->nx * p->ny * p->nz <= GRAPH_AUTO_CELLS;
}

// A graph exec that advances `steps` (even) steps from blocks (a, b) - or, in
// place (b == NULL), from representation `repr` of block a.  NULL if the capture
// cannot be done (the caller then launches directly).
cudaGraphExec_t graph_for(mlb_plan *p, void *a, void *b, int steps, int repr)
{
    mlb_plan::GraphCache &gc = p->gc;
    if (gc.exec && gc.a == a && gc.b == b && gc.epoch == p->epoch && gc.steps == steps
        && gc.repr == repr)
        return gc.exec;
    if (gc.exec) {
        cudaGraphExecDestroy(gc.exec);
        gc.exec = nullptr;
    }
    if (!p->cap_stream
        && cudaStreamCreateWithFlags(&p->cap_stream, cudaStreamNonBlocking) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    if (cudaStreamBeginCapture(p->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    const long long launches0 = g_launches.load();
    int rc = MLB_OK;
    if (b) {
        void *pre = a, *post = b;
        for (int t = 0; t < steps && rc == MLB_OK; ++t) {
            rc = one_step(p, pre, post, p->cap_stream);
            void *tmp = pre; pre = post; post = tmp;
        }
    } else {
        int r = repr;
        for (int t = 0; t < steps && rc == MLB_OK; ++t, r ^= 1)
            rc = launch_aa_any(p, a, r, p->cap_stream);
    }
    const long long nodes = g_launches.load() - launches0;
    g_launches.fetch_sub(nodes);   // captured, not launched: replays are counted
    cudaGraph_t graph = nullptr;
    const cudaError_t e = cudaStreamEndCapture(p->cap_stream, &graph);
    if (rc != MLB_OK || e != cudaSuccess || !graph) {
        (void)cudaGetLastError();
        if (graph) cudaGraphDestroy(graph);
        return nullptr;
    }
    cudaGraphExec_t exec = nullptr;
    if (cudaGraphInstantiate(&exec, graph, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        exec = nullptr;
    }
    cudaGraphDestroy(graph);
    if (exec) {
        gc.exec = exec; gc.a = a; gc.b = b; gc.epoch = p->epoch; gc.steps = steps;
        gc.repr = repr; gc.nodes = nodes;
    }
    return exec;
}

// replays of a captured run; returns the number of steps done (a multiple of 2,
// so blocks / representation are back where they started)
int run_graphed(mlb_plan *p, void *a, void *b, int nsteps, int repr, cudaStream_t st, int *done)
{
    *done = 0;
    if (!graph_wanted(p, nsteps))
        return MLB_OK;
    const int unit = nsteps >= GRAPH_STEPS ? GRAPH_STEPS : (nsteps & ~1);
    cudaGraphExec_t exec = graph_for(p, a, b, unit, repr);
    if (!exec)
        return MLB_OK;
    for (int n = nsteps / unit; n > 0; --n) {
        MLB_CUDA(cudaGraphLaunch(exec, st));
        g_launches.fetch_add(p->gc.nodes, std::memory_order_relaxed);
        *done += unit;
    }
    return MLB_OK;
}

}  // namespace

int mlb_plan_set_inplace_layout(mlb_plan *p, int mode)
{
    if (int rc = check_plan(p, false)) return rc;
    if (mode < -1 || mode > 1)
        return fail(MLB_EINVAL, "in-place layout %d: must be -1 (auto), 0 (classic) or 1 (row blocks)", mode);
    p->aa_layout = mode;
    ++p->epoch;
    return MLB_OK;
}

int mlb_plan_set_graph(mlb_plan *p, int mode)
{
    if (int rc = check_plan(p, false)) return rc;
    if (mode < -1 || mode > 1)
        return fail(MLB_EINVAL, "graph mode %d: must be -1 (auto), 0 (never) or 1 (always)", mode);
    p->graph_mode = mode;
    return MLB_OK;
}

int mlb_run_steps(mlb_plan *p, void *d_a, void *d_b, int nsteps, void *stream, float *ms)
{
    if (int rc = check_plan(p, true)) return rc;
    if (p->z_mode != MLB_Z_PERIODIC)
        return fail(MLB_EUNSUPPORTED, "mlb_run_steps needs an MLB_Z_PERIODIC plan; a slab's "
                    "halo exchange happens between steps (mlb_slab_run_steps)");
    if (nsteps < 0) return fail(MLB_EINVAL, "nsteps < 0");
    if (!d_a || !d_b) return fail(MLB_EINVAL, "NULL population block");
    if (d_a == d_b) return fail(MLB_EINVAL, "fpre and fpost must be distinct blocks");
    MLB_ON_DEVICE(p->device);
    if (ms) MLB_CUDA(cudaEventRecord(p->ev0, S(stream)));
    int done = 0;
    if (int rc = run_graphed(p, d_a, d_b, nsteps, 0, S(stream), &done)) return rc;
    void *pre = d_a, *post = d_b;   // `done` is even: the blocks are where they started
    for (int t = done; t < nsteps; ++t) {
        if (int rc = one_step(p, pre, post, stream)) return rc;
        void *tmp = pre; pre = post; post = tmp;
    }
    if (ms) {
        MLB_CUDA(cudaEventRecord(p->ev1, S(stream)));
        MLB_CUDA(cudaEventSynchronize(p->ev1));
        MLB_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
    }
    return MLB_OK;
}

static int check_inplace(const mlb_plan *p, const void *d_f, const int *repr)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_f || !repr) return fail(MLB_EINVAL, "NULL argument");
    if (*repr != 0 && *repr != 1)
        return fail(MLB_EINVAL, "representation must be 0 (normal) or 1 (shifted), got %d", *repr);
    if (p->z_mode != MLB_Z_PERIODIC)
        return fail(MLB_EUNSUPPORTED, "the in-place update needs an MLB_Z_PERIODIC plan "
                    "(whole domain on one GPU)");
    if (!aa_open_ok(p, resolve_aa_variant(p)))
        return fail(MLB_EUNSUPPORTED, "the in-place update handles walls only unless a pack "
                    "kernel runs (variant W*1000 + LX, or auto with "
                    "nx >= 128) and every outlet cell has its x-1 neighbour in the same pack; this "
                    "geometry has %lld inlet and %lld outlet cells - use the two-buffer path",
                    p->n_in, p->n_out);
    return MLB_OK;
}

int mlb_run_steps_inplace(mlb_plan *p, void *d_f, int nsteps, int *repr, void *stream, float *ms)
{
    if (int rc = check_inplace(p, d_f, repr)) return rc;
    if (nsteps < 0) return fail(MLB_EINVAL, "nsteps < 0");
    MLB_ON_DEVICE(p->device);
    if (ms) MLB_CUDA(cudaEventRecord(p->ev0, S(stream)));
    int done = 0;
    if (int rc = run_graphed(p, d_f, nullptr, nsteps, *repr, S(stream), &done)) return rc;
    for (int t = done; t < nsteps; ++t) {
        if (int rc = launch_aa_any(p, d_f, *repr, S(stream))) return rc;
        *repr ^= 1;
    }
    if (ms) {
        MLB_CUDA(cudaEventRecord(p->ev1, S(stream)));
        MLB_CUDA(cudaEventSynchronize(p->ev1));
        MLB_CUDA(cudaEventElapsedTime(ms, p->ev0, p->ev1));
    }
    return MLB_OK;
}

int mlb_inplace_normalize(mlb_plan *p, void *d_f, int *repr, void *stream)
{
    if (int rc = check_inplace(p, d_f, repr)) return rc;
    if (*repr == 0) return MLB_OK;
    MLB_ON_DEVICE(p->device);
    if (int rc = launch_aa_any(p, d_f, 2, S(stream))) return rc;
    *repr = 0;
    return MLB_OK;
}

int mlb_step_inplace_range(mlb_plan *p, void *d_f, int repr, int z0, int z1, void *d_below,
                           int nz_below, void *d_above, int nz_above, void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_f) return fail(MLB_EINVAL, "NULL population block");
    if (repr != 0 && repr != 1)
        return fail(MLB_EINVAL, "representation must be 0 (normal) or 1 (shifted), got %d", repr);
    if (z0 < 0 || z1 > p->nz || z0 > z1)
        return fail(MLB_EINVAL, "plane range [%d, %d) outside [0, %d)", z0, z1, p->nz);
    if (p->z_mode != MLB_Z_HALO)
        return fail(MLB_EUNSUPPORTED, "mlb_step_inplace_range is the z-slab form (MLB_Z_HALO "
                    "plans); a whole domain uses mlb_run_steps_inplace");
    if (!d_below || !d_above || nz_below < 1 || nz_above < 1)
        return fail(MLB_EINVAL, "the in-place slab step needs both ring neighbours' blocks "
                    "(with one slab: the block itself)");
    const int variant = resolve_aa_variant(p);
    if (!aa_uses_packs(p, variant))
        return fail(MLB_EUNSUPPORTED, "the in-place slab step needs a pack kernel (variant "
                    "W*1000 + LX, or auto with nx >= 128)");
    if (!aa_open_ok(p, variant))
        return fail(MLB_EUNSUPPORTED, "the in-place update handles walls only unless every outlet "
                    "cell has its x-1 neighbour in the same pack; this geometry has %lld inlet "
                    "and %lld outlet cells", p->n_in, p->n_out);
    if (z0 == z1) return MLB_OK;
    MLB_ON_DEVICE(p->device);
    AaRange r;
    r.z0 = z0; r.z1 = z1;
    r.below = d_below; r.nz_below = nz_below;
    r.above = d_above; r.nz_above = nz_above;
    return launch_aa_any(p, d_f, repr, S(stream), r);
}

int mlb_inplace_swap_slab(mlb_plan *p, void *d_f, void *d_above, int nz_above, void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_f || !d_above || nz_above < 1) return fail(MLB_EINVAL, "NULL / empty block");
    if (p->z_mode != MLB_Z_HALO)
        return fail(MLB_EUNSUPPORTED, "mlb_inplace_swap_slab is the z-slab form; a whole domain "
                    "uses mlb_inplace_normalize");
    MLB_ON_DEVICE(p->device);
    AaRange r;
    r.above = d_above; r.nz_above = nz_above;
    return launch_aa_any(p, d_f, 2, S(stream), r);
}

// 5 crossing populations of one boundary plane of a slab with src_nz planes
// into a halo plane of a slab with dst_nz planes (same plane shape, dtype).
static int halo_copy_impl(const mlb_plan *p, void *d_dst, int dst_nz, const void *d_src,
                          int src_nz, int face, cudaStream_t st)
{
    const long long plane = p->lay.plane;
    const long long src_pop = (long long)(src_nz + 2) * plane;
    const long long dst_pop = (long long)(dst_nz + 2) * plane;
    mlb::HaloArgs h;
    for (int j = 0; j < 5; ++j) {
        const int q = face == 0 ? mlb::halo_up(j) : mlb::halo_down(j);
        h.src_off[j] = q * src_pop + (face == 0 ? (long long)src_nz : 1LL) * plane;
        h.dst_off[j] = q * dst_pop + (face == 0 ? 0LL : (long long)(dst_nz + 1)) * plane;
    }
    h.words = plane * p->lay.itemsize / 16;
    const dim3 grid((unsigned)((h.words + 255) / 256), 5);
    mlb::halo_copy_kernel<<<grid, 256, 0, st>>>(d_src, d_dst, h, p->lay.itemsize);
    MLB_LAUNCHED();
    return MLB_OK;
}

int mlb_halo_copy(const mlb_plan *p, void *d_dst, const void *d_src, int src_nz, int face,
                  void *stream)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!d_dst || !d_src) return fail(MLB_EINVAL, "NULL population block");
    if (src_nz < 1 || (face != 0 && face != 1))
        return fail(MLB_EINVAL, "bad src_nz %d / face %d", src_nz, face);
    MLB_ON_DEVICE(p->device);
    return halo_copy_impl(p, d_dst, p->nz, d_src, src_nz, face, S(stream));
}

int mlb_halo_push(const mlb_plan *p, const void *d_src, void *d_dst, int dst_nz, int face,
                  void *stream)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!d_dst || !d_src) return fail(MLB_EINVAL, "NULL population block");
    if (dst_nz < 1 || (face != 0 && face != 1))
        return fail(MLB_EINVAL, "bad dst_nz %d / face %d", dst_nz, face);
    MLB_ON_DEVICE(p->device);
    return halo_copy_impl(p, d_dst, dst_nz, d_src, p->nz, face, S(stream));
}

int mlb_step_push_range(mlb_plan *p, const void *d_fpre, void *d_fpost, int z0, int z1,
                        void *d_below_post, int nz_below, void *d_above_post, int nz_above,
                        void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_fpre || !d_fpost) return fail(MLB_EINVAL, "NULL population block");
    if (d_fpre == d_fpost)
        return fail(MLB_EINVAL, "fpre and fpost must be distinct blocks");
    if (z0 < 0 || z1 > p->nz || z0 > z1)
        return fail(MLB_EINVAL, "plane range [%d, %d) outside [0, %d)", z0, z1, p->nz);
    if ((d_below_post && nz_below < 1) || (d_above_post && nz_above < 1))
        return fail(MLB_EINVAL, "neighbour slab plane counts must be >= 1");
    if (d_below_post == d_fpre || d_above_post == d_fpre)
        return fail(MLB_EINVAL, "a push target is the block this step reads");
    if (z0 == z1) return MLB_OK;
    // only a launch that covers a boundary plane has anything to push
    PushTarget t;
    if (z0 == 0 && d_below_post) { t.below = d_below_post; t.nz_below = nz_below; }
    if (z1 == p->nz && d_above_post) { t.above = d_above_post; t.nz_above = nz_above; }
    const bool any = t.below || t.above;
    MLB_ON_DEVICE(p->device);
    const bool open_cells = p->in_zoff[z1] > p->in_zoff[z0] || p->out_zoff[z1] > p->out_zoff[z0];
    const bool fuse = can_fuse_open(p, resolve_variant(p, !any));   // the kernel launch_step picks
    if (!open_cells || fuse)
        return launch_step(p, d_fpre, d_fpost, z0, z1, S(stream), fuse, any ? &t : nullptr);
    // list-driven open-boundary pass: it rewrites cells of the boundary plane
    // after the fused kernel, so the plane is pushed afterwards, as a copy
    if (int rc = launch_step(p, d_fpre, d_fpost, z0, z1, S(stream))) return rc;
    if (int rc = mlb_open_pass_range(p, d_fpost, z0, z1, stream)) return rc;
    if (t.above)
        if (int rc = halo_copy_impl(p, t.above, t.nz_above, d_fpost, p->nz, 0, S(stream))) return rc;
    if (t.below)
        if (int rc = halo_copy_impl(p, t.below, t.nz_below, d_fpost, p->nz, 1, S(stream))) return rc;
    return MLB_OK;
}

// ---- the z-slab time-step loop, one call ---------------------------------------
// What slab.DistSlab schedules per step, without a host interpreter in the loop:
//   main:  record fork                         interior planes [1, nz-1)   wait join
//   hi:    wait fork, wait both counters >= t-1, plane 0 (+ push down),
//          plane nz-1 (+ push up), post t into both neighbours, record join
extern "C++" {
namespace {

int check_ring(const mlb_plan *p, const mlb_ring *r, int nblocks)
{
    if (!r) return fail(MLB_EINVAL, "ring is NULL");
    for (int k = 0; k < nblocks; ++k)
        if (!r->below[k] || !r->above[k])
            return fail(MLB_EINVAL, "ring: neighbour block %d is NULL", k);
    if (r->nz_below < 1 || r->nz_above < 1)
        return fail(MLB_EINVAL, "ring: neighbour slab plane counts must be >= 1");
    if (!r->post_below || !r->post_above || !r->wait_below || !r->wait_above)
        return fail(MLB_EINVAL, "ring: NULL signal slot");
    if (r->wait_mode < 0 || r->wait_mode > 2)
        return fail(MLB_EINVAL, "ring: wait mode must be 0 (auto), 1 or 2");
    if (p->z_mode != MLB_Z_HALO)
        return fail(MLB_EUNSUPPORTED, "the slab loop needs an MLB_Z_HALO plan");
    return MLB_OK;
}

struct HostClock {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double us() const
    {
        return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
            .count();
    }
};

// one step of the schedule; `boundary(z0, z1, st)` / `interior(st)` enqueue the launches
template <typename FB, typename FI>
int slab_step(mlb_plan *p, mlb_ring *r, cudaStream_t main, cudaStream_t hi, FB boundary,
              FI interior)
{
    const uint32_t t = r->t + 1;
    const bool overlap = r->overlap && p->nz >= 3 && hi != nullptr && hi != main;
    cudaStream_t bs = overlap ? hi : main;
    if (overlap) {
        MLB_CUDA(cudaEventRecord(p->ev_fork, main));
        MLB_CUDA(cudaStreamWaitEvent(hi, p->ev_fork, 0));
    }
    if (int rc = mlb_signal_wait(r->wait_below, t - 1, r->wait_mode, bs)) return rc;
    if (int rc = mlb_signal_wait(r->wait_above, t - 1, r->wait_mode, bs)) return rc;
    if (overlap) {
        if (int rc = boundary(0, 1, bs)) return rc;
        if (int rc = boundary(p->nz - 1, p->nz, bs)) return rc;
    } else {
        if (int rc = boundary(0, p->nz, bs)) return rc;
    }
    if (int rc = mlb_signal_post(r->post_below, t, bs)) return rc;
    if (int rc = mlb_signal_post(r->post_above, t, bs)) return rc;
    r->t = t;
    if (overlap) {
        if (int rc = interior(main)) return rc;
        MLB_CUDA(cudaEventRecord(p->ev_join, hi));
        MLB_CUDA(cudaStreamWaitEvent(main, p->ev_join, 0));
    }
    return MLB_OK;
}

}  // namespace
}  // extern "C++"

int mlb_slab_run_steps(mlb_plan *p, void *d_a, void *d_b, int nsteps, mlb_ring *ring,
                       void *stream, void *hi_stream, double *host_us)
{
    if (int rc = check_plan(p, true)) return rc;
    if (int rc = check_ring(p, ring, 2)) return rc;
    if (!d_a || !d_b || d_a == d_b) return fail(MLB_EINVAL, "need two distinct population blocks");
    if (nsteps < 0) return fail(MLB_EINVAL, "nsteps < 0");
    MLB_ON_DEVICE(p->device);
    void *blk[2] = {d_a, d_b};
    HostClock clock;
    double first = 0.0;
    int counted = 0;
    for (int s = 0; s < nsteps; ++s) {
        const int ipre = s & 1, ipost = ipre ^ 1;
        void *pre = blk[ipre], *post = blk[ipost];
        auto boundary = [&](int z0, int z1, cudaStream_t st) {
            return mlb_step_push_range(p, pre, post, z0, z1, ring->below[ipost], ring->nz_below,
                                       ring->above[ipost], ring->nz_above, st);
        };
        auto interior = [&](cudaStream_t st) {
            return mlb_step_open_range(p, pre, post, 1, p->nz - 1, st);
        };
        if (int rc = slab_step(p, ring, S(stream), S(hi_stream), boundary, interior)) return rc;
        if (s < 32) { first = clock.us(); counted = s + 1; }   // before the launch queue can fill
    }
    if (host_us) *host_us = counted ? first / counted : 0.0;
    return MLB_OK;
}

int mlb_slab_run_steps_inplace(mlb_plan *p, void *d_f, int nsteps, int *repr, mlb_ring *ring,
                               void *stream, void *hi_stream, double *host_us)
{
    if (int rc = check_plan(p, true)) return rc;
    if (int rc = check_ring(p, ring, 1)) return rc;
    if (!d_f || !repr) return fail(MLB_EINVAL, "NULL argument");
    if (*repr != 0 && *repr != 1)
        return fail(MLB_EINVAL, "representation must be 0 (normal) or 1 (shifted), got %d", *repr);
    if (nsteps < 0) return fail(MLB_EINVAL, "nsteps < 0");
    MLB_ON_DEVICE(p->device);
    HostClock clock;
    double first = 0.0;
    int counted = 0;
    for (int s = 0; s < nsteps; ++s) {
        const int rp = *repr;
        auto boundary = [&](int z0, int z1, cudaStream_t st) {
            return mlb_step_inplace_range(p, d_f, rp, z0, z1, ring->below[0], ring->nz_below,
                                          ring->above[0], ring->nz_above, st);
        };
        auto interior = [&](cudaStream_t st) {
            return mlb_step_inplace_range(p, d_f, rp, 1, p->nz - 1, ring->below[0],
                                          ring->nz_below, ring->above[0], ring->nz_above, st);
        };
        if (int rc = slab_step(p, ring, S(stream), S(hi_stream), boundary, interior)) return rc;
        *repr ^= 1;
        if (s < 32) { first = clock.us(); counted = s + 1; }
    }
    if (host_us) *host_us = counted ? first / counted : 0.0;
    return MLB_OK;
}

int mlb_macro(const mlb_plan *p, const void *d_f, double *d_rho, double *d_ux, double *d_uy,
              double *d_uz, void *stream)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!d_f || !d_rho || !d_ux || !d_uy || !d_uz) return fail(MLB_EINVAL, "NULL buffer");
    MLB_ON_DEVICE(p->device);
    // (the diagnostics read storage only: mixed2 - float in memory - shares the float kernels)
    const int V = p->dtype == MLB_F64 ? 2 : 4;   // cells per pack (16 / 16 / 8 bytes)
    if (p->nx % V == 0) {
        const dim3 grid((p->nx / V + 127) / 128, p->ny, p->nz);
        if (p->dtype == MLB_F32 || p->dtype == MLB_F32C64)
            mlb::macro_vec_kernel<float, 4><<<grid, 128, 0, S(stream)>>>(
                static_cast<const float *>(d_f), p->g, d_rho, d_ux, d_uy, d_uz);
        else if (p->dtype == MLB_F64)
            mlb::macro_vec_kernel<double, 2><<<grid, 128, 0, S(stream)>>>(
                static_cast<const double *>(d_f), p->g, d_rho, d_ux, d_uy, d_uz);
        else
            mlb::macro_vec_kernel<__half, 4><<<grid, 128, 0, S(stream)>>>(
                static_cast<const __half *>(d_f), p->g, d_rho, d_ux, d_uy, d_uz);
        MLB_LAUNCHED();
        return MLB_OK;
    }
    const dim3 grid((p->nx + 127) / 128, p->ny, p->nz);
    if (p->dtype == MLB_F32 || p->dtype == MLB_F32C64)
        mlb::macro_kernel<float><<<grid, 128, 0, S(stream)>>>(
            static_cast<const float *>(d_f), p->g, d_rho, d_ux, d_uy, d_uz);
    else if (p->dtype == MLB_F64)
        mlb::macro_kernel<double><<<grid, 128, 0, S(stream)>>>(
            static_cast<const double *>(d_f), p->g, d_rho, d_ux, d_uy, d_uz);
    else
        mlb::macro_kernel<__half><<<grid, 128, 0, S(stream)>>>(
            static_cast<const __half *>(d_f), p->g, d_rho, d_ux, d_uy, d_uz);
    MLB_LAUNCHED();
    return MLB_OK;
}

int mlb_diagnostics(mlb_plan *p, const void *d_f, double h_out[8], void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!d_f || !h_out) return fail(MLB_EINVAL, "NULL buffer");
    MLB_ON_DEVICE(p->device);
    const bool packs = p->nx % (p->dtype == MLB_F64 ? 2 : 4) == 0;
    const mlb::ClsTab ct = cls_tab(p);
    const int nb = p->diag_blocks, nt = mlb::DIAG_THREADS;
    if (p->dtype == MLB_F32 || p->dtype == MLB_F32C64) {
        const float *f = static_cast<const float *>(d_f);
        if (packs) mlb::diag_vec_kernel<float, 4, false><<<nb, nt, 0, S(stream)>>>(f, ct, p->g, p->d_partials);
        else mlb::diag_kernel<float, 1><<<nb, nt, 0, S(stream)>>>(f, ct, p->g, p->d_partials);
    } else if (p->dtype == MLB_F64) {
        const double *f = static_cast<const double *>(d_f);
        if (packs) mlb::diag_vec_kernel<double, 2, true><<<nb, nt, 0, S(stream)>>>(f, ct, p->g, p->d_partials);
        else mlb::diag_kernel<double, 2><<<nb, nt, 0, S(stream)>>>(f, ct, p->g, p->d_partials);
    } else {
        const __half *f = static_cast<const __half *>(d_f);
        if (packs) mlb::diag_vec_kernel<__half, 4, true><<<nb, nt, 0, S(stream)>>>(f, ct, p->g, p->d_partials);
        else mlb::diag_kernel<__half, 1><<<nb, nt, 0, S(stream)>>>(f, ct, p->g, p->d_partials);
    }
    MLB_LAUNCHED();
    mlb::diag_final_kernel<<<1, mlb::DIAG_THREADS, 0, S(stream)>>>(p->d_partials,
                                                                  p->diag_blocks, p->d_diag);
    MLB_LAUNCHED();
    MLB_CUDA(cudaMemcpyAsync(h_out, p->d_diag, sizeof(double) * mlb::DIAG_N,
                             cudaMemcpyDeviceToHost, S(stream)));
    MLB_CUDA(cudaStreamSynchronize(S(stream)));
    return MLB_OK;
}

int mlb_probe(const mlb_plan *p, const void *d_f, int x, int y, int lz, double *d_out4,
              void *stream)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!d_f || !d_out4) return fail(MLB_EINVAL, "NULL buffer");
    if (x < 0 || x >= p->nx || y < 0 || y >= p->ny || lz < 0 || lz >= p->nz)
        return fail(MLB_EINVAL, "probe cell (%d, %d, %d) outside the slab", x, y, lz);
    MLB_ON_DEVICE(p->device);
    if (p->dtype == MLB_F32 || p->dtype == MLB_F32C64)
        mlb::probe_kernel<float><<<1, 1, 0, S(stream)>>>(static_cast<const float *>(d_f),
                                                         p->g, x, y, lz, d_out4);
    else if (p->dtype == MLB_F64)
        mlb::probe_kernel<double><<<1, 1, 0, S(stream)>>>(static_cast<const double *>(d_f),
                                                          p->g, x, y, lz, d_out4);
    else
        mlb::probe_kernel<__half><<<1, 1, 0, S(stream)>>>(static_cast<const __half *>(d_f),
                                                          p->g, x, y, lz, d_out4);
    MLB_LAUNCHED();
    return MLB_OK;
}

int mlb_step_host(mlb_plan *p, const void *h_fpre, void *h_fpost, void *d_a, void *d_b,
                  void *stream)
{
    if (int rc = check_plan(p, true)) return rc;
    if (!h_fpre || !h_fpost || !d_a || !d_b) return fail(MLB_EINVAL, "NULL buffer");
    if (h_fpre == h_fpost)
        return fail(MLB_EINVAL, "fpre and fpost must be distinct blocks");
    if (p->z_mode != MLB_Z_PERIODIC)
        return fail(MLB_EUNSUPPORTED, "mlb_step_host needs an MLB_Z_PERIODIC plan");
    if (int rc = mlb_upload(p, h_fpre, d_a, stream)) return rc;
    if (int rc = mlb_upload(p, h_fpost, d_b, stream)) return rc;
    if (int rc = mlb_step(p, d_a, d_b, stream)) return rc;
    if (int rc = mlb_download(p, d_b, h_fpost, stream)) return rc;
    MLB_CUDA(cudaStreamSynchronize(S(stream)));
    return MLB_OK;
}

// ---- a whole run on HOST blocks, transfers overlapped with the steps ------------
// engine.run on a host-resident state (engine.py:218-275) is upload, K steps,
// download; at PCIe speed the two transfers of a 512^3 fp32 block take 0.19 s
// each, the 20 steps between them 0.06 s.  When the domain is closed in z (planes
// 0 and nz-1 are walls: no update depends on the periodic wrap) the three phases
// can overlap.  The domain is cut into chunks of z planes and the steps are
// time-skewed: step s of chunk c runs at tick c + s, right after step s-1 of
// chunk c+1 (same stream, so the planes it still reads in the block it will
// overwrite have been consumed).  Chunk u is uploaded at tick u on a copy
// stream; chunk c's final populations are downloaded on a second copy stream
// as soon as its last step is done - while later chunks are still arriving
// (PCIe is full duplex).  Every cell sees exactly the launches of the plain
// loop restricted to its plane range, so the result is the plain loop's, bit
// for bit.  At most SKEW_MAX steps ride on each transfer (the kernels must keep
// up with the link); the steps in between run as plain whole-domain launches.
namespace {

constexpr int SKEW_MAX = 40;

struct ChunkCopy {
    const mlb_plan *p;
    int z0, z1;
    // one strided copy for all 19 populations when rows are not padded
    cudaError_t run(void *dst, const void *src, cudaMemcpyKind kind, cudaStream_t st) const
    {
        const int sz = p->lay.itemsize;
        const size_t row = (size_t)p->nx * sz, rows = (size_t)(z1 - z0) * p->ny;
        const size_t dense_pop = (size_t)p->nz * p->ny * row;
        const size_t dev_pop = (size_t)p->lay.pop * sz, dev_row = (size_t)p->lay.xp * sz;
        const size_t hoff = (size_t)z0 * p->ny * row, doff = ((size_t)z0 + 1) * p->lay.plane * sz;
        const bool h2d = kind == cudaMemcpyHostToDevice, d2d = kind == cudaMemcpyDeviceToDevice;
        if (d2d)
            return cudaMemcpy2DAsync((char *)dst + doff, dev_pop, (const char *)src + doff, dev_pop,
                                     rows * dev_row, MLB_Q, kind, st);
        if (p->lay.xp == p->nx)
            return h2d ? cudaMemcpy2DAsync((char *)dst + doff, dev_pop, (const char *)src + hoff,
                                           dense_pop, rows * row, MLB_Q, kind, st)
                       : cudaMemcpy2DAsync((char *)dst + hoff, dense_pop, (const char *)src + doff,
                                           dev_pop, rows * row, MLB_Q, kind, st);
        for (int q = 0; q < MLB_Q; ++q) {
            const cudaError_t e =
                h2d ? cudaMemcpy2DAsync((char *)dst + q * dev_pop + doff, dev_row,
                                        (const char *)src + q * dense_pop + hoff, row, row, rows,
                                        kind, st)
                    : cudaMemcpy2DAsync((char *)dst + q * dense_pop + hoff, row,
                                        (const char *)src + q * dev_pop + doff, dev_row, row, rows,
                                        kind, st);
            if (e != cudaSuccess) return e;
        }
        return cudaSuccess;
    }
};

}  // namespace

int mlb_run_steps_host(mlb_plan *p, const void *h_in, void *h_out, void *d_a, void *d_b,
                       int nsteps, int chunk_planes, const uint8_t *h_flags, void *stream,
                       float *ms, int *overlapped)
{
    if (int rc = check_plan(p, false)) return rc;
    if (!h_in || !h_out || !d_a || !d_b || d_a == d_b)
        return fail(MLB_EINVAL, "need host source / destination and two distinct device blocks");
    if (nsteps < 0) return fail(MLB_EINVAL, "nsteps < 0");
    if (p->z_mode != MLB_Z_PERIODIC)
        return fail(MLB_EUNSUPPORTED, "mlb_run_steps_host needs an MLB_Z_PERIODIC plan");
    if (!p->have_flags && !h_flags)
        return fail(MLB_EINVAL, "plan has no flags and none were passed");
    MLB_ON_DEVICE(p->device);
    cudaStream_t cs = S(stream);
    if (!p->up_stream) MLB_CUDA(cudaStreamCreateWithFlags(&p->up_stream, cudaStreamNonBlocking));
    if (!p->down_stream) MLB_CUDA(cudaStreamCreateWithFlags(&p->down_stream, cudaStreamNonBlocking));
    const int nz = p->nz;
    int cz = chunk_planes > 0 ? (chunk_planes < nz ? chunk_planes : nz) : (nz + 127) / 128;
    // automatic choice: a chunk of a population should stay at least 1 MB (copy efficiency)
    while (chunk_planes <= 0 && cz < nz && (size_t)cz * p->lay.plane * p->lay.itemsize < (1u << 20))
        ++cz;
    const int C = (nz + cz - 1) / cz;
    auto zlo = [&](int c) { return c * cz; };
    auto zhi = [&](int c) { return (c + 1) * cz < nz ? (c + 1) * cz : nz; };

    if (ms) MLB_CUDA(cudaEventRecord(p->ev0, cs));
    // The flag tables first.  (Enqueuing the uploads first and building the tables
    // "meanwhile" does not work: the flag copy queues behind every chunk already
    // handed to the copy engine, and the first kernel would wait for the whole
    // upload - measured 0.40 s instead of 0.27 s for 20 steps at 512^3.)
    if (!p->have_flags)
        if (int rc = mlb_plan_set_flags(p, h_flags, nullptr, nullptr)) return rc;
    std::vector<cudaEvent_t> up(C, nullptr), done(C, nullptr);
    auto cleanup = [&]() {
        for (cudaEvent_t e : up) if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : done) if (e) cudaEventDestroy(e);
    };
#define MLB_CUDA_C(expr)                                                        \
    do {                                                                        \
        cudaError_t e_ = (expr);                                                \
        if (e_ != cudaSuccess) {                                                \
            cleanup();                                                          \
            return fail(MLB_ECUDA, "%s: %s (%s:%d)", #expr,                     \
                        cudaGetErrorString(e_), __FILE__, __LINE__);            \
        }                                                                       \
    } while (0)
    // (the copy stream starts after whatever the caller enqueued before)
    MLB_CUDA_C(cudaEventRecord(p->ev_fork, cs));
    MLB_CUDA_C(cudaStreamWaitEvent(p->up_stream, p->ev_fork, 0));
    MLB_CUDA_C(cudaStreamWaitEvent(p->down_stream, p->ev_fork, 0));
    for (int c = 0; c < C; ++c) {
        MLB_CUDA_C(cudaEventCreateWithFlags(&up[c], cudaEventDisableTiming));
        MLB_CUDA_C(cudaEventCreateWithFlags(&done[c], cudaEventDisableTiming));
        const ChunkCopy cc{p, zlo(c), zhi(c)};
        MLB_CUDA_C(cc.run(d_a, h_in, cudaMemcpyHostToDevice, p->up_stream));
        MLB_CUDA_C(cudaEventRecord(up[c], p->up_stream));
    }
    // both blocks identical from here on (engine.py:148): pass-through stores are valid
    // unless the geometry chains outlet cells
    p->passthrough = p->out_chained ? 0 : 1;
    ++p->epoch;

    const bool skew = p->z_closed && C >= 4 && nsteps >= 1;
    if (overlapped) *overlapped = skew ? 1 : 0;
    void *blk[2] = {d_a, d_b};
    int rc = MLB_OK;
    auto download = [&](int c, void *src) -> cudaError_t {
        cudaError_t e = cudaEventRecord(done[c], cs);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(p->down_stream, done[c], 0);
        if (e == cudaSuccess)
            e = ChunkCopy{p, zlo(c), zhi(c)}.run(h_out, src, cudaMemcpyDeviceToHost, p->down_stream);
        return e;
    };
    // one time-skewed sweep of `S` steps starting from block `from`; uploads ride on
    // it when `with_up`, downloads when `with_down`
    auto sweep = [&](int S, int from, bool with_up, bool with_down) -> int {
        for (int u = 0; u < C + S; ++u) {
            if (with_up && u < C) {
                MLB_CUDA(cudaStreamWaitEvent(cs, up[u], 0));
                MLB_CUDA((ChunkCopy{p, zlo(u), zhi(u)}.run(d_b, d_a, cudaMemcpyDeviceToDevice, cs)));
            }
            for (int s = 1; s <= S; ++s) {
                const int c = u - s;
                if (c < 0 || c >= C) continue;
                void *pre = blk[(from + s - 1) & 1], *post = blk[(from + s) & 1];
                if (int r = mlb_step_open_range(p, pre, post, zlo(c), zhi(c), stream)) return r;
                if (s == S && with_down) MLB_CUDA(download(c, post));
            }
        }
        return MLB_OK;
    };
    if (skew) {
        const int s1 = nsteps < SKEW_MAX ? nsteps : SKEW_MAX;
        const int rest = nsteps - s1;
        const int s3 = rest < SKEW_MAX ? rest : SKEW_MAX, s2 = rest - s3;
        rc = sweep(s1, 0, true, rest == 0);
        int at = s1 & 1;
        for (int t = 0; t < s2 && rc == MLB_OK; ++t, at ^= 1)
            rc = one_step(p, blk[at], blk[at ^ 1], stream);
        if (rc == MLB_OK && s3 > 0) rc = sweep(s3, at, false, true);
    } else {
        // no overlap possible (periodic in z, or a tiny domain): the plain sequence
        for (int c = 0; c < C && rc == MLB_OK; ++c) {
            cudaError_t e = cudaStreamWaitEvent(cs, up[c], 0);
            if (e == cudaSuccess)
                e = ChunkCopy{p, zlo(c), zhi(c)}.run(d_b, d_a, cudaMemcpyDeviceToDevice, cs);
            if (e != cudaSuccess) rc = fail(MLB_ECUDA, "chunk copy: %s", cudaGetErrorString(e));
        }
        int at = 0;
        for (int t = 0; t < nsteps && rc == MLB_OK; ++t, at ^= 1)
            rc = one_step(p, blk[at], blk[at ^ 1], stream);
        for (int c = 0; c < C && rc == MLB_OK; ++c) {
            const cudaError_t e = download(c, blk[at]);
            if (e != cudaSuccess) rc = fail(MLB_ECUDA, "download: %s", cudaGetErrorString(e));
        }
    }
    if (rc == MLB_OK) {
        // join: the caller's stream ends after the last download
        cudaError_t e = cudaEventRecord(p->ev_join, p->down_stream);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, p->ev_join, 0);
        if (e == cudaSuccess && ms) e = cudaEventRecord(p->ev1, cs);
        if (e == cudaSuccess) e = cudaStreamSynchronize(cs);
        if (e == cudaSuccess && ms) e = cudaEventElapsedTime(ms, p->ev0, p->ev1);
        if (e != cudaSuccess) rc = fail(MLB_ECUDA, "mlb_run_steps_host: %s", cudaGetErrorString(e));
    } else {
        cudaDeviceSynchronize();
    }
    cleanup();
#undef MLB_CUDA_C
    return rc;
}

// ---- peer memory: CUDA IPC mapping and stream-ordered signals --------------
namespace {

// driver entry points, resolved at run time (the library does not link libcuda,
// so it still loads - and exports every symbol - on a box without a driver)
typedef int (*cuStreamWaitValue32_t)(cudaStream_t, unsigned long long, unsigned int, unsigned int);
typedef int (*cuMemGetAddressRange_t)(unsigned long long *, size_t *, unsigned long long);

void *driver_entry(const char *name)
{
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess
        || q != cudaDriverEntryPointSuccess)
        return nullptr;
    return fn;
}

__global__ void signal_post_kernel(volatile unsigned int *slot, unsigned int value)
{
    // everything earlier on this stream (the boundary kernel's stores into the
    // neighbour's halo) is ordered before the flag, system-wide
    __threadfence_system();
    *slot = value;
}

__global__ void signal_wait_kernel(const volatile unsigned int *slot, unsigned int value)
{
    // *slot >= value, wrap-around safe
    while ((int)(*slot - value) < 0)
        __nanosleep(200);
    __threadfence_system();
}

}  // namespace

int mlb_ipc_export(const void *d_ptr, unsigned char handle[MLB_IPC_HANDLE_BYTES],
                   int64_t *offset)
{
    static_assert(sizeof(cudaIpcMemHandle_t) == MLB_IPC_HANDLE_BYTES, "IPC handle size");
    if (!d_ptr || !handle || !offset) return fail(MLB_EINVAL, "NULL argument");
    // the handle names the whole allocation; find its base (torch sub-allocates)
    static cuMemGetAddressRange_t range = (cuMemGetAddressRange_t)driver_entry("cuMemGetAddressRange");
    unsigned long long base = (unsigned long long)(uintptr_t)d_ptr;
    size_t size = 0;
    if (range) {
        const int rc = range(&base, &size, (unsigned long long)(uintptr_t)d_ptr);
        if (rc != 0)
            return fail(MLB_ECUDA, "cuMemGetAddressRange failed (%d): not a device allocation?", rc);
    }
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void *)(uintptr_t)base);
    if (e != cudaSuccess)
        return fail(MLB_ECUDA, "cudaIpcGetMemHandle: %s (blocks must come from cudaMalloc - "
                    "torch's default allocator does; expandable_segments / cudaMallocAsync "
                    "pools do not)", cudaGetErrorString(e));
    std::memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((unsigned long long)(uintptr_t)d_ptr - base);
    return MLB_OK;
}

int mlb_ipc_open(int device, const unsigned char handle[MLB_IPC_HANDLE_BYTES], void **d_base)
{
    if (!handle || !d_base) return fail(MLB_EINVAL, "NULL argument");
    MLB_ON_DEVICE(device);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    MLB_CUDA(cudaIpcOpenMemHandle(d_base, h, cudaIpcMemLazyEnablePeerAccess));
    return MLB_OK;
}

int mlb_ipc_close(void *d_base)
{
    if (!d_base) return MLB_OK;
    MLB_CUDA(cudaIpcCloseMemHandle(d_base));
    return MLB_OK;
}

int mlb_signal_create(int device, void **d_sig)
{
    if (!d_sig) return fail(MLB_EINVAL, "NULL argument");
    MLB_ON_DEVICE(device);
    MLB_CUDA(g_pool.alloc(d_sig, MLB_SIGNAL_BYTES));
    MLB_CUDA(cudaMemset(*d_sig, 0, MLB_SIGNAL_BYTES));
    MLB_CUDA(cudaDeviceSynchronize());
    return MLB_OK;
}

int mlb_signal_destroy(void *d_sig)
{
    if (d_sig) MLB_CUDA(cudaDeviceSynchronize());
    pool_free(d_sig);
    return MLB_OK;
}

int mlb_signal_post(void *d_slot, uint32_t value, void *stream)
{
    if (!d_slot) return fail(MLB_EINVAL, "NULL slot");
    signal_post_kernel<<<1, 1, 0, S(stream)>>>(static_cast<volatile unsigned int *>(d_slot), value);
    MLB_LAUNCHED();
    return MLB_OK;
}

int mlb_signal_wait(const void *d_slot, uint32_t value, int mode, void *stream)
{
    if (!d_slot) return fail(MLB_EINVAL, "NULL slot");
    if (mode < 0 || mode > 2) return fail(MLB_EINVAL, "wait mode must be 0 (auto), 1 or 2");
    static cuStreamWaitValue32_t wait32 = (cuStreamWaitValue32_t)driver_entry("cuStreamWaitValue32");
    if (mode != 2 && wait32) {
        // CU_STREAM_WAIT_VALUE_GEQ = 0: the stream stalls in the front end, no SM is held
        const int rc = wait32(S(stream), (unsigned long long)(uintptr_t)d_slot, value, 0u);
        if (rc == 0) return MLB_OK;
        if (mode == 1) return fail(MLB_ECUDA, "cuStreamWaitValue32 failed (%d)", rc);
    } else if (mode == 1) {
        return fail(MLB_EUNSUPPORTED, "cuStreamWaitValue32 is not available from this driver");
    }
    signal_wait_kernel<<<1, 1, 0, S(stream)>>>(static_cast<const volatile unsigned int *>(d_slot),
                                                 value);
    MLB_LAUNCHED();
    return MLB_OK;
}

int mlb_trim(void)
{
    g_pool.trim();
    g_blocks.trim();
    return MLB_OK;
}

int mlb_block_alloc(int device, int64_t bytes, void **d_out)
{
    if (!d_out) return fail(MLB_EINVAL, "NULL argument");
    *d_out = nullptr;
    if (bytes <= 0) return fail(MLB_EINVAL, "block of %lld bytes", (long long)bytes);
    int ndev = 0;
    MLB_CUDA(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return fail(MLB_EINVAL, "device %d out of range (%d visible)", device, ndev);
    MLB_ON_DEVICE(device);
    cudaError_t e = g_blocks.alloc(d_out, (size_t)bytes);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        g_pool.trim();                 // the plans' idle tables too, then once more
        e = g_blocks.alloc(d_out, (size_t)bytes);
    }
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        return fail(MLB_ENOMEM, "cudaMalloc of a %.2f GB population block on device %d: %s",
                    (double)bytes / 1e9, device, cudaGetErrorString(e));
    }
    return MLB_OK;
}

int mlb_block_free(void *d_ptr)
{
    if (!d_ptr) return MLB_OK;
    cudaPointerAttributes at;
    int dev = -1;
    if (cudaPointerGetAttributes(&at, d_ptr) == cudaSuccess && at.type == cudaMemoryTypeDevice)
        dev = at.device;
    else
        (void)cudaGetLastError();
    if (dev < 0) return fail(MLB_EINVAL, "not a device allocation");
    MLB_ON_DEVICE(dev);
    // a pooled block may be handed to the next caller at once: whatever still
    // uses it must be over (the wait cudaFree implies)
    MLB_CUDA(cudaDeviceSynchronize());
    g_blocks.release(d_ptr);
    return MLB_OK;
}

int mlb_signal_wait_kind(void)
{
    static const bool memop = driver_entry("cuStreamWaitValue32") != nullptr;
    return memop ? 1 : 2;
}

int mlb_signal_read(const void *d_slot, uint32_t *out)
{
    if (!d_slot || !out) return fail(MLB_EINVAL, "NULL argument");
    MLB_CUDA(cudaMemcpy(out, d_slot, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    return MLB_OK;
}

}  // extern "C"
