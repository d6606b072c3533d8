// Achievable HBM bandwidth for the PCG update's access mix on this B200:
// read x, p, r, ap, pre (5 streams), write x, r (2 streams), N doubles each.
#include <cstdio>
#include <cuda_runtime.h>
template <int U>
__global__ void upd(int n, double a, double *x, const double *p, double *r, const double *ap, const double *pre, double *out) {
    double s = 0;
    const int stride = gridDim.x * blockDim.x * U;
    for (int i0 = blockIdx.x * blockDim.x * U + threadIdx.x; i0 < n; i0 += stride) {
        double xv[U], pv[U], rv[U], av[U], dv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) { int i = i0 + u * blockDim.x; if (i < n) { xv[u] = x[i]; pv[u] = p[i]; rv[u] = r[i]; av[u] = ap[i]; dv[u] = pre[i]; } }
#pragma unroll
        for (int u = 0; u < U; ++u) { int i = i0 + u * blockDim.x; if (i < n) { x[i] = xv[u] + a * pv[u]; double rr = rv[u] - a * av[u]; r[i] = rr; s += rr * dv[u] * rr; } }
    }
    if (s == 1234.5) out[0] = s;
}
__global__ void copyk(int n, const double *a, double *b) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
    const int n = 3835221; int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *v[8]; for (auto &q : v) { cudaMalloc(&q, n * 8); cudaMemset(q, 0, n * 8); }
    double *flush; size_t fb = 512ull << 20; cudaMalloc(&flush, fb);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
    auto run = [&](const char *name, auto launch, double bytes) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(flush, rep, fb);
            cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        printf("{\"kernel\":\"%s\",\"us\":%.1f,\"GBps\":%.0f}\n", name, best * 1e3, bytes / best / 1e6);
    };
    const double ub = 7.0 * n * 8;
    for (int ctas : {sms * 4, sms * 8, sms * 16}) {
        char nm[64];
        snprintf(nm, 64, "upd_u1_%d", ctas); run(nm, [&] { upd<1><<<ctas, 256>>>(n, 0.5, v[0], v[1], v[2], v[3], v[4], v[7]); }, ub);
        snprintf(nm, 64, "upd_u4_%d", ctas); run(nm, [&] { upd<4><<<ctas, 256>>>(n, 0.5, v[0], v[1], v[2], v[3], v[4], v[7]); }, ub);
    }
    run("copy", [&] { copyk<<<sms * 8, 256>>>(n, v[5], v[6]); }, 2.0 * n * 8);
    return 0;
}
