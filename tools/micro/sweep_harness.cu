// Development harness: runs ONE dumped NVRTC sweep kernel (QF_JIT_DUMP) in
// isolation on a hash-filled n = 30 complex64 state pair and checks a few tiles
// against a host restatement of that sweep (the last adjoint sweep of HEA D=1,
// n = 30: cx(0,1); TY tap + ry(0); TZ tap + rz(1); TY tap + ry(1)).
//   nvcc -std=c++17 -O2 -gencode arch=compute_100a,code=sm_100a -DGEN_SRC='"path.cu"' sweep_harness.cu
#include GEN_SRC
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <complex>

using namespace qfb;
typedef std::complex<double> cd;

__host__ __device__ inline float hashf(uint64_t i, uint32_t salt) {
    uint64_t x = i * 0x9E3779B97F4A7C15ull + salt;
    x ^= x >> 31; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 29;
    return (float)((double)(x >> 40) / (double)(1ull << 24) - 0.5);
}
__global__ void fill(float2* p, uint64_t n, uint32_t salt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = make_float2(hashf(i, salt), hashf(i, salt + 7));
}

int main() {
    const int n = 30;
    const uint64_t N = 1ull << n;
    float2 *psi, *lam, *gmat;
    double* tap;
    const int ntiles = 1 << 18, ntaps = 60;
    if (cudaMalloc(&psi, N * 8) || cudaMalloc(&lam, N * 8) || cudaMalloc(&tap, (size_t)ntaps * ntiles * 8) ||
        cudaMalloc(&gmat, 120 * 8)) { printf("alloc failed\n"); return 1; }
    fill<<<4096, 256>>>(psi, N, 1);
    fill<<<4096, 256>>>(lam, N, 2);
    // gmat block (offset 114): ry(0) shear (t, s), rz(1) d0 d1, ry(1) shear
    const double th0 = 0.7, th1 = -1.3, ph = 0.4;
    auto shear = [](double th) { double s = std::sin(th / 2), c = std::cos(th / 2); return std::make_pair(s / (1 + c), s); };
    // adjoint shear = rotation by -theta
    auto s0 = shear(-th0), s1 = shear(-th1);
    std::vector<float2> hg(120, make_float2(0, 0));
    hg[114] = make_float2((float)s0.first, (float)s0.second);
    hg[116] = make_float2((float)std::cos(ph / 2), (float)(std::sin(ph / 2)));   // conj(e^{-i ph/2})
    hg[117] = make_float2((float)std::cos(ph / 2), (float)(-std::sin(ph / 2)));  // conj(e^{+i ph/2})
    hg[118] = make_float2((float)s1.first, (float)s1.second);
    cudaMemcpy(gmat, hg.data(), 120 * 8, cudaMemcpyHostToDevice);
    SweepArgs a{};
    a.psi = psi; a.lam = lam; a.n = n; a.tap_part = tap; a.n_taps_total = ntaps;
    a.gmat = gmat; a.gmat_stride = 120; a.gmat_pass_base = 0; a.batch = 1;
    const size_t smem = 65536 + 48 + 3 * 256 * 4;
    cudaFuncSetAttribute(qf_sweep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    qf_sweep<<<dim3(ntiles, 1), 256, smem>>>(a);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    // host check of a few tiles: tile bits = 0..9, 28, 29; tile_base = tile_id << 10
    const double u_re = std::cos(ph), u_im = std::sin(ph);  // d1 conj(d0) for rz(ph)^dagger = e^{-i ph}?  sign checked below
    int bad = 0;
    for (uint32_t tid_ : {0u, 1u, 77777u, (uint32_t)ntiles - 1}) {
        const uint64_t base = (uint64_t)tid_ << 10;
        std::vector<cd> x(4096), y(4096);
        auto mem = [&](int l) { return base | (uint64_t)(l & 1023) | ((uint64_t)(l >> 10) << 28); };  // l: bits 0-9 low, 10 -> 28, 11 -> 29
        for (int l = 0; l < 4096; ++l) {
            x[l] = cd(hashf(mem(l), 1), hashf(mem(l), 8));
            y[l] = cd(hashf(mem(l), 2), hashf(mem(l), 9));
        }
        const int B28 = 1 << 10, B29 = 1 << 11;
        // cx(0,1): control bit 29, target bit 28
        for (int l = 0; l < 4096; ++l)
            if ((l & B29) && !(l & B28)) { std::swap(x[l], x[l | B28]); std::swap(y[l], y[l | B28]); }
        double taps[3] = {0, 0, 0};
        auto ty = [&](int B) {
            double s = 0;
            for (int l = 0; l < 4096; ++l)
                if (!(l & B)) s += (std::conj(y[l | B]) * x[l]).real() - (std::conj(y[l]) * x[l | B]).real();
            return s;
        };
        auto rot = [&](int B, double th) {  // R_y(th) on pairs
            const double c = std::cos(th / 2), s = std::sin(th / 2);
            for (int l = 0; l < 4096; ++l)
                if (!(l & B)) {
                    cd a0 = x[l], a1 = x[l | B]; x[l] = c * a0 - s * a1; x[l | B] = s * a0 + c * a1;
                    a0 = y[l]; a1 = y[l | B]; y[l] = c * a0 - s * a1; y[l | B] = s * a0 + c * a1;
                }
        };
        taps[0] = ty(B29);
        rot(B29, -th0);
        double tz = 0;
        for (int l = 0; l < 4096; ++l) tz += ((l & B28) ? -1 : 1) * (std::conj(y[l]) * x[l]).imag();
        taps[1] = tz;
        const cd u = cd(std::cos(ph / 2), -std::sin(ph / 2)) * std::conj(cd(std::cos(ph / 2), std::sin(ph / 2)));
        for (int l = 0; l < 4096; ++l)
            if (l & B28) { x[l] *= u; y[l] *= u; }
        taps[2] = ty(B28);
        rot(B28, -th1);
        (void)u_re; (void)u_im;
        // device results
        double maxd = 0, maxa = 0;
        for (int l = 0; l < 4096; l += 1) {
            float2 gx, gy;
            cudaMemcpy(&gx, psi + mem(l), 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&gy, lam + mem(l), 8, cudaMemcpyDeviceToHost);
            maxd = std::max(maxd, std::abs(cd(gx.x, gx.y) - x[l]) + std::abs(cd(gy.x, gy.y) - y[l]));
            maxa = std::max(maxa, std::abs(x[l]));
            if (std::abs(cd(gx.x, gx.y) - x[l]) > 1e-4 && bad < 8) {
                ++bad;
                printf("  tile %u l=%d (bits28,29=%d%d, low=%d): dev (%g,%g) host (%g,%g)\n", tid_, l, (l >> 10) & 1,
                       (l >> 11) & 1, l & 1023, gx.x, gx.y, x[l].real(), x[l].imag());
            }
        }
        double dt[3];
        for (int t = 0; t < 3; ++t) cudaMemcpy(&dt[t], tap + (size_t)(57 + t) * ntiles + tid_, 8, cudaMemcpyDeviceToHost);
        printf("tile %u: max|d state| %.3e (max|amp| %.3e)  taps dev %.6e %.6e %.6e host %.6e %.6e %.6e\n", tid_, maxd, maxa,
               dt[0], dt[1], dt[2], taps[0], taps[1], taps[2]);
    }
    return 0;
}
