// Exact last stage (exact_last_stage=True): the 3-D
// non-equispaced DFT of the trig-polynomial coefficients eta on I_n^3 at the
// warped nodes, and its adjoint, by direct summation on the device.
//
// Reference: nfft.py:51-82 (ndft / ndft_adjoint), used by transform.py:393-394
// (forward) and :404-405 (adjoint).  eta lives in the plan's "grid" buffer
// with N = n (no oversampling, no halo) in FFT order: frequency k on axis j
// at index k mod n_j.  O(M n0 n1 n2): a verification mode for small problems.
#include "sgl_internal.cuh"

namespace sgl {
namespace {

// f_i = sum_k eta[k] e^{+i k . tau_i}; one warp per node, lanes over k2
__global__ void k_ndft_fwd(int64_t M, NodeSet nodes, int n0, int n1, int n2, const double2 *__restrict__ eta,
                           double2 *__restrict__ out) {
    const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= M) return;
    const double t0 = nodes.u0[i] * (kTwoPi / n0), t1 = nodes.u1[i] * (kTwoPi / n1), t2 = nodes.u2[i] * (kTwoPi / n2);
    double ar = 0.0, ai = 0.0;
    for (int p0 = 0; p0 < n0; ++p0) {
        const int k0 = p0 - n0 / 2;
        double s0, c0;
        sincos(k0 * t0, &s0, &c0);
        for (int p1 = 0; p1 < n1; ++p1) {
            const int k1 = p1 - n1 / 2;
            double s1, c1;
            sincos(k1 * t1, &s1, &c1);
            const double er = c0 * c1 - s0 * s1, ei = c0 * s1 + s0 * c1;
            const double2 *row = eta + ((size_t)((k0 + n0) % n0) * n1 + (k1 + n1) % n1) * n2;
            double sr = 0.0, si = 0.0;
            for (int p2 = lane; p2 < n2; p2 += 32) {
                const int k2 = p2 - n2 / 2;
                double s2, c2;
                sincos(k2 * t2, &s2, &c2);
                const double2 v = row[(k2 + n2) % n2];
                sr += v.x * c2 - v.y * s2;
                si += v.x * s2 + v.y * c2;
            }
            ar += er * sr - ei * si;
            ai += er * si + ei * sr;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ar += __shfl_xor_sync(0xffffffffu, ar, o);
        ai += __shfl_xor_sync(0xffffffffu, ai, o);
    }
    if (lane == 0) out[nodes.perm[i]] = make_double2(ar, ai);
}

// eta_t[k] = sum_i v_i e^{-i k . tau_i}; one block per (k0, k1), threads over k2
__global__ void k_ndft_adj(int64_t M, NodeSet nodes, int n0, int n1, int n2, const double2 *__restrict__ values,
                           double2 *__restrict__ eta) {
    const int p0 = blockIdx.x / n1, p1 = blockIdx.x % n1;
    const int k0 = p0 - n0 / 2, k1 = p1 - n1 / 2;
    for (int p2 = threadIdx.x; p2 < n2; p2 += blockDim.x) {
        const int k2 = p2 - n2 / 2;
        double ar = 0.0, ai = 0.0;
        for (int64_t i = 0; i < M; ++i) {
            const double ph = k0 * (nodes.u0[i] * (kTwoPi / n0)) + k1 * (nodes.u1[i] * (kTwoPi / n1)) +
                              k2 * (nodes.u2[i] * (kTwoPi / n2));
            double s, c;
            sincos(ph, &s, &c);
            const double2 v = values[nodes.perm[i]];
            ar += v.x * c + v.y * s;   // v * e^{-i ph}
            ai += v.y * c - v.x * s;
        }
        eta[((size_t)((k0 + n0) % n0) * n1 + (k1 + n1) % n1) * n2 + (k2 + n2) % n2] = make_double2(ar, ai);
    }
}

}  // namespace

int launch_exact_forward(const Plan &p, const double2 *eta, double2 *values, cudaStream_t st) {
    if (p.M == 0) return SGL_OK;
    const int64_t threads = p.M * 32;
    k_ndft_fwd<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(p.M, p.nodes, p.grid[0], p.grid[1], p.grid[2], eta,
                                                                  values);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

int launch_exact_adjoint(const Plan &p, const double2 *values, double2 *eta, cudaStream_t st) {
    k_ndft_adj<<<(unsigned)(p.grid[0] * p.grid[1]), 128, 0, st>>>(p.M, p.nodes, p.grid[0], p.grid[1], p.grid[2],
                                                                  values, eta);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

}  // namespace sgl
