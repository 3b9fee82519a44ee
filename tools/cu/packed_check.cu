// Does the packed-fp32 collide (Alg<float2>) produce the same bits as the scalar one?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o packed_check packed_check.cu
#include "../../paper_2409_16781_b200/csrc/mlb_kernels.cuh"
#include <cstdio>
#include <cstring>
#include <vector>
using namespace mlb;

#define NREC 64
template <typename L>
__device__ void collide_rec(L (&g)[Q], const typename Alg<L>::S omega_, L *rec)
{
    using A = Alg<L>;
    using S = typename A::S;
    int r = 0;
#define REC(x) rec[r++] = (x)
    const L one = A::cst(S(1.0)), omega = A::cst(omega_);
    const L c3 = A::cst(S(3.0)), c45 = A::cst(S(4.5)), c15 = A::cst(S(1.5));
    const L w0 = A::cst(S(1.0 / 3.0)), ws = A::cst(S(1.0 / 18.0)), wd = A::cst(S(1.0 / 36.0));
    L rho = A::add(g[0], g[1]);
#pragma unroll
    for (int i = 2; i < Q; ++i) rho = A::add(rho, g[i]);
    REC(rho);
    const L mx = A::add(A::sub(A::sub(A::add(A::add(A::sub(A::sub(A::add(A::sub(
        g[1], g[3]), g[5]), g[6]), g[7]), g[8]), g[11]), g[12]), g[13]), g[14]);
    const L my = A::add(A::sub(A::sub(A::add(A::sub(A::sub(A::add(A::add(A::sub(
        g[2], g[4]), g[5]), g[6]), g[7]), g[8]), g[15]), g[16]), g[17]), g[18]);
    const L mz = A::sub(A::sub(A::add(A::add(A::sub(A::sub(A::add(A::add(A::sub(
        g[9], g[10]), g[11]), g[12]), g[13]), g[14]), g[15]), g[16]), g[17]), g[18]);
    REC(mx); REC(my); REC(mz);
    const L inv = A::rcp0(rho); REC(inv);
    const L ux = A::mul(mx, inv), uy = A::mul(my, inv), uz = A::mul(mz, inv);
    REC(ux); REC(uy); REC(uz);
    const L usq = A::add(A::add(A::mul(ux, ux), A::mul(uy, uy)), A::mul(uz, uz)); REC(usq);
    const L um = A::sub(one, A::mul(c15, usq)); REC(um);
    const L wr0 = A::mul(w0, rho), wrs = A::mul(ws, rho), wrd = A::mul(wd, rho);
    REC(wr0); REC(wrs); REC(wrd);
    const L a = A::add(ux, uy), b = A::sub(ux, uy), c = A::add(ux, uz), d = A::sub(ux, uz),
            h = A::add(uy, uz), kk = A::sub(uy, uz);
    REC(a); REC(b); REC(c); REC(d); REC(h); REC(kk);
#define PAIR(cu, wr, ip, im) { \
        const L q_ = A::mul(c45, A::mul((cu), (cu))); REC(q_); \
        const L t_ = A::mul(c3, (cu)); REC(t_); \
        const L p_ = A::add(um, q_); REC(p_); \
        const L ep_ = A::mul((wr), A::add(p_, t_)); REC(ep_); \
        const L em_ = A::mul((wr), A::sub(p_, t_)); REC(em_); \
        g[ip] = A::sub(g[ip], A::mul(omega, A::sub(g[ip], ep_))); \
        g[im] = A::sub(g[im], A::mul(omega, A::sub(g[im], em_))); }
    PAIR(ux, wrs, 1, 3) PAIR(uy, wrs, 2, 4) PAIR(a, wrd, 5, 7) PAIR(b, wrd, 8, 6)
    PAIR(uz, wrs, 9, 10) PAIR(c, wrd, 11, 13) PAIR(d, wrd, 14, 12) PAIR(h, wrd, 15, 17)
    PAIR(kk, wrd, 18, 16)
    { const L e0 = A::mul(wr0, um); REC(e0); g[0] = A::sub(g[0], A::mul(omega, A::sub(g[0], e0))); }
}

__global__ void check(const float *in, int ncells, float omega, float *out_s, float *out_p,
                      float *rec_s, float *rec_p)
{
    const int pair = blockIdx.x * blockDim.x + threadIdx.x;
    if (2 * pair + 1 >= ncells) return;
    float gs0[Q], gs1[Q]; float2 gp[Q];
    for (int i = 0; i < Q; ++i) {
        gs0[i] = in[(2 * pair) * Q + i]; gs1[i] = in[(2 * pair + 1) * Q + i];
        gp[i] = make_float2(gs0[i], gs1[i]);
    }
    float r0[NREC], r1[NREC]; float2 rp[NREC];
    for (int i = 0; i < NREC; ++i) { r0[i] = r1[i] = 0.f; rp[i] = make_float2(0.f, 0.f); }
    collide_rec<float>(gs0, omega, r0);
    collide_rec<float>(gs1, omega, r1);
    collide_rec<float2>(gp, omega, rp);
    for (int i = 0; i < Q; ++i) {
        out_s[(2 * pair) * Q + i] = gs0[i]; out_s[(2 * pair + 1) * Q + i] = gs1[i];
        out_p[(2 * pair) * Q + i] = gp[i].x; out_p[(2 * pair + 1) * Q + i] = gp[i].y;
    }
    for (int i = 0; i < NREC; ++i) {
        rec_s[(2 * pair) * NREC + i] = r0[i]; rec_s[(2 * pair + 1) * NREC + i] = r1[i];
        rec_p[(2 * pair) * NREC + i] = rp[i].x; rec_p[(2 * pair + 1) * NREC + i] = rp[i].y;
    }
}

int main()
{
    const int n = 1 << 20;
    std::vector<float> in((size_t)n * Q);
    unsigned long long s = 88172645463325252ull;
    for (auto &v : in) {
        s ^= s << 13; s ^= s >> 7; s ^= s << 17;
        // half-precision-representable inputs in (0.02, 1), like the failing test
        float u = 0.02f + 0.98f * (float)((s >> 11) * (1.0 / 9007199254740992.0));
        v = __half2float(__float2half_rn(u));
    }
    float *d_in, *d_s, *d_p, *d_rs, *d_rp;
    cudaMalloc(&d_in, in.size() * 4); cudaMalloc(&d_s, in.size() * 4); cudaMalloc(&d_p, in.size() * 4);
    cudaMalloc(&d_rs, (size_t)n * NREC * 4); cudaMalloc(&d_rp, (size_t)n * NREC * 4);
    cudaMemcpy(d_in, in.data(), in.size() * 4, cudaMemcpyHostToDevice);
    check<<<n / 2 / 128, 128>>>(d_in, n, 1.45f, d_s, d_p, d_rs, d_rp);
    std::vector<float> os(in.size()), op(in.size()), rs((size_t)n * NREC), rp((size_t)n * NREC);
    cudaMemcpy(os.data(), d_s, os.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(op.data(), d_p, op.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(rs.data(), d_rs, rs.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(rp.data(), d_rp, rp.size() * 4, cudaMemcpyDeviceToHost);
    printf("cuda: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    long bad = 0, shown = 0;
    for (int c = 0; c < n; ++c) {
        bool diff = memcmp(&os[(size_t)c * Q], &op[(size_t)c * Q], Q * 4) != 0;
        if (!diff) continue;
        ++bad;
        if (shown++ < 3) {
            printf("cell %d differs; first differing intermediates:\n", c);
            int k = 0;
            for (int i = 0; i < NREC && k < 4; ++i)
                if (memcmp(&rs[(size_t)c * NREC + i], &rp[(size_t)c * NREC + i], 4)) {
                    printf("  rec[%d]: scalar %.9g (%08x) packed %.9g (%08x)\n", i, rs[(size_t)c * NREC + i],
                           *(unsigned *)&rs[(size_t)c * NREC + i], rp[(size_t)c * NREC + i],
                           *(unsigned *)&rp[(size_t)c * NREC + i]);
                    ++k;
                }
            for (int i = 0; i < Q; ++i)
                if (memcmp(&os[(size_t)c * Q + i], &op[(size_t)c * Q + i], 4))
                    printf("  out[%d]: scalar %.9g packed %.9g  (g_in %.9g)\n", i, os[(size_t)c * Q + i],
                           op[(size_t)c * Q + i], in[(size_t)c * Q + i]);
        }
    }
    printf("cells with differing float results: %ld of %d\n", bad, n);
    return 0;
}
