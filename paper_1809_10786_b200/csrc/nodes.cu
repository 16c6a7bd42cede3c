// Plan-time node processing on the device: radius check, warp to torus
// coordinates, pencil/lo0 sort and greedy window tiles.
//
// Follows transform.py:39-55 (choose_rho, transform_points) and
// nfft.py:131-133, 177-178 (reduction into [0, 2pi), u = N tau / 2 pi,
// lo = floor(u)) of the reference.  The sort and the tiles have no
// reference counterpart (the reference walks nodes unsorted).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "i8_common.cuh"
#include "sgl_internal.cuh"

namespace sgl {

namespace {

__global__ void k_check_radius(const double *pts, int64_t M, double limit, int *bad) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < M) {
        double r = pts[3 * i];
        if (!(r <= limit)) atomicOr(bad, 1);  // NaN counts as bad too
    }
}

__global__ void k_radius(const double *pts, int64_t M, double *r) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < M) r[i] = pts[3 * i];
}

__device__ __forceinline__ double reduce_2pi(double x) {
    // np.mod(x, 2 pi) with the 2 pi -> 0 fold of nfft.py:177-178
    double t = fmod(x, kTwoPi);
    if (t < 0.0) t += kTwoPi;
    if (t >= kTwoPi) t = 0.0;
    return t;
}

__device__ __forceinline__ void to_u(double tau, int N, double &u, int &lo) {
    u = (double)N * tau / kTwoPi;     // nfft.py:132 evaluation order
    double f = floor(u);
    lo = (int)f;
    if (lo >= N) {                    // rounding onto N: same cell modulo N
        u -= (double)N;
        lo -= N;
    }
}

// plain NFFT nodes: already on the torus (nfft.py:177-178, 131-133)
// (m, d) rows; the leading 3 - d axes are length-1 dummies at 0
__global__ void k_torus(const double *pts, int64_t M, int d, int N0, int N1, int N2, double *u0, double *u1,
                        double *u2) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    double *us[3] = {u0, u1, u2};
    const int Ns[3] = {N0, N1, N2};
    for (int ax = 0; ax < 3; ++ax) {
        int l;
        if (ax < 3 - d)
            us[ax][i] = 0.0;
        else
            to_u(reduce_2pi(pts[d * i + ax - (3 - d)]), Ns[ax], us[ax][i], l);
    }
}

struct KeyGeom {
    int N0, N1, N2, W1, W2, P2;   // pencils of W1 x W2 cells on axes 1-2, P2 per row
    uint64_t line_base;           // first key of the grid-line nodes (see k_key)
    int q;                        // window half-width (grid-line test)
};

__global__ void k_warp(const double *pts, int64_t M, double rho, int N0, int N1, int N2, double *u0,
                       double *u1, double *u2) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    double r = pts[3 * i], th = pts[3 * i + 1], ph = pts[3 * i + 2];
    double gam = (2.0 * r - rho) / rho;                 // transform.py:52
    gam = fmin(1.0, fmax(-1.0, gam));
    double t0 = reduce_2pi(acos(gam));
    double t1 = reduce_2pi(th);
    double t2 = reduce_2pi(ph);
    double a, b, c;
    int l0, l1, l2;
    to_u(t0, N0, a, l0);
    to_u(t1, N1, b, l1);
    to_u(t2, N2, c, l2);
    u0[i] = a;
    u1[i] = b;
    u2[i] = c;
}

__global__ void k_key(const double *u0, const double *u1, const double *u2, int64_t M, KeyGeom g, uint64_t *key,
                      int32_t *idx) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    const double v1 = u1[i], v2 = u2[i];
    const int l0 = (int)floor(u0[i]), l1 = (int)floor(v1), l2 = (int)floor(v2);
    // A node on (or within rounding of) a grid line of axis 1 or 2 has 2q+1 taps there, so in
    // a W-wide pencil its box would exceed the device slab and cut the tile
    // short (structured inputs: config 2's lattice puts ~2 % of its nodes on
    // the phi = k pi/2 and theta = pi/2 planes).  Such nodes get their own
    // single-cell pencils after all regular ones.
    int c1lo, c1hi, c2lo, c2hi;
    window_cells(v1, g.q, c1lo, c1hi);
    window_cells(v2, g.q, c2lo, c2hi);
    if (g.line_base && (c1hi - c1lo == 2 * g.q || c2hi - c2lo == 2 * g.q)) {
        key[i] = g.line_base + ((uint64_t)l1 * (uint64_t)g.N2 + (uint64_t)l2) * (uint64_t)g.N0 + (uint64_t)l0;
    } else {
        const uint64_t pencil = (uint64_t)(l1 / g.W1) * (uint64_t)g.P2 + (uint64_t)(l2 / g.W2);
        key[i] = pencil * (uint64_t)g.N0 + (uint64_t)l0;
    }
    idx[i] = (int32_t)i;
}

__global__ void k_permute(const int32_t *idx, int64_t M, const double *a0, const double *a1,
                          const double *a2, double *b0, double *b1, double *b2) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    int32_t j = idx[i];
    b0[i] = a0[j];
    b1[i] = a1[j];
    b2[i] = a2[j];
}

__global__ void k_run_heads(const uint64_t *key, int64_t M, uint64_t N0, int32_t *head) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    head[i] = (i == 0 || key[i] / N0 != key[i - 1] / N0) ? 1 : 0;
}

__global__ void k_run_starts(const int32_t *head, const int32_t *rank, int64_t M, int32_t *starts) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= M) return;
    if (head[i]) starts[rank[i]] = (int32_t)i;
}

struct TileGeom {
    int q;
    int span0;      // max lo0 span inside a tile
    int max_nodes;  // nodes per tile
    int box0;       // max box extent on axis 0
    int box1 = kBoxMax, box2 = kBoxMax;   // max box extents on axes 1-2
};

__device__ __forceinline__ int lo_of(double u) { return (int)floor(u); }

// One thread per pencil run: greedy cut into tiles of <= max_nodes nodes
// whose lo0 span is <= span0.  write == nullptr: count only.
__global__ void k_tiles(const int32_t *starts, int64_t nruns, int64_t M, const double *u0,
                        const double *u1, const double *u2, TileGeom g, int32_t *counts,
                        const int32_t *offsets, Tile *out) {
    int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nruns) return;
    int64_t s = starts[r];
    int64_t e = (r + 1 < nruns) ? starts[r + 1] : M;
    int32_t nt = 0;
    int64_t pos = out ? offsets[r] : 0;
    int64_t i = s;
    while (i < e) {
        int first0 = lo_of(u0[i]);
        int mn[3] = {1 << 30, 1 << 30, 1 << 30}, mx[3] = {-(1 << 30), -(1 << 30), -(1 << 30)};
        int64_t j = i;
        for (; j < e && j - i < g.max_nodes; ++j) {
            double uu[3] = {u0[j], u1[j], u2[j]};
            int l0 = lo_of(uu[0]);
            if (l0 - first0 > g.span0) break;
            int tmn[3], tmx[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                int c_lo, c_hi;   // the reference's taps: 2q+1 on (or within rounding of) a grid line, else 2q
                window_cells(uu[d], g.q, c_lo, c_hi);
                tmn[d] = min(mn[d], c_lo);
                tmx[d] = max(mx[d], c_hi);
            }
            // the box must fit the device slab (axes 1, 2) and the slab-count limit (axis 0)
            if (j > i && (tmx[1] - tmn[1] + 1 > g.box1 || tmx[2] - tmn[2] + 1 > g.box2 ||
                          tmx[0] - tmn[0] + 1 > g.box0))
                break;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                mn[d] = tmn[d];
                mx[d] = tmx[d];
            }
        }
        if (out) {
            Tile t;
            t.start = (int32_t)i;
            t.count = (int32_t)(j - i);
            t.o0 = mn[0];
            t.o1 = mn[1];
            t.o2 = mn[2];
            t.e0 = mx[0] - mn[0] + 1;
            t.e1 = mx[1] - mn[1] + 1;
            t.e2 = mx[2] - mn[2] + 1;
            out[pos++] = t;
        }
        ++nt;
        i = j;
    }
    if (!out) counts[r] = nt;
}

// plan-time scratch from the stream-ordered pool (cudaMallocAsync): frees do
// not synchronise the device
thread_local cudaStream_t t_plan_stream = nullptr;

// One warp per pencil run: the same greedy cut as k_tiles (tiles of <=
// max_nodes nodes, lo0 span <= span0, box within the slab limits), 32 nodes
// per step: per-lane window cells, warp prefix min / max of the box, and the
// first lane that fails ends the tile.  write == nullptr: count only.
__global__ void k_tiles_warp(const int32_t *starts, int64_t nruns, int64_t M, const double *u0, const double *u1,
                             const double *u2, TileGeom g, int32_t *counts, const int32_t *offsets, Tile *out) {
    const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= nruns) return;
    const int64_t s = starts[r];
    const int64_t e = (r + 1 < nruns) ? starts[r + 1] : M;
    int32_t nt = 0;
    int64_t pos = out ? offsets[r] : 0;
    int64_t i = s;
    const int BIG = 1 << 30;
    while (i < e) {
        const int first0 = lo_of(u0[i]);
        int mn[3] = {BIG, BIG, BIG}, mx[3] = {-BIG, -BIG, -BIG};
        int64_t j = i;
        for (;;) {
            const int64_t k = j + lane;
            const bool valid = k < e && k - i < g.max_nodes;
            int cl[3] = {BIG, BIG, BIG}, ch[3] = {-BIG, -BIG, -BIG};
            bool fail = !valid;
            if (valid) {
                const double uu[3] = {u0[k], u1[k], u2[k]};
                if (lo_of(uu[0]) - first0 > g.span0) fail = true;
#pragma unroll
                for (int d = 0; d < 3; ++d) window_cells(uu[d], g.q, cl[d], ch[d]);
            }
            // inclusive prefix min / max over the lanes, merged with the tile so far
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const int a = __shfl_up_sync(0xffffffffu, cl[d], o), b = __shfl_up_sync(0xffffffffu, ch[d], o);
                    if (lane >= o) {
                        cl[d] = min(cl[d], a);
                        ch[d] = max(ch[d], b);
                    }
                }
            }
            int tmn[3], tmx[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                tmn[d] = min(mn[d], cl[d]);
                tmx[d] = max(mx[d], ch[d]);
            }
            if (valid && k > i &&
                (tmx[1] - tmn[1] + 1 > g.box1 || tmx[2] - tmn[2] + 1 > g.box2 || tmx[0] - tmn[0] + 1 > g.box0))
                fail = true;
            const unsigned bad = __ballot_sync(0xffffffffu, fail);
            const int take = bad ? __ffs(bad) - 1 : 32;   // accepted lanes of this step
            if (take > 0) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    mn[d] = __shfl_sync(0xffffffffu, tmn[d], take - 1);
                    mx[d] = __shfl_sync(0xffffffffu, tmx[d], take - 1);
                }
            }
            j += take;
            if (take < 32) break;
        }
        if (out && lane == 0) {
            Tile t;
            t.start = (int32_t)i;
            t.count = (int32_t)(j - i);
            t.o0 = mn[0];
            t.o1 = mn[1];
            t.o2 = mn[2];
            t.e0 = mx[0] - mn[0] + 1;
            t.e1 = mx[1] - mn[1] + 1;
            t.e2 = mx[2] - mn[2] + 1;
            out[pos] = t;
        }
        ++pos;
        ++nt;
        i = j;
    }
    if (!out && lane == 0) counts[r] = nt;
}

template <typename T>
struct DevBuf {
    T *p = nullptr;
    cudaStream_t st = t_plan_stream;
    ~DevBuf() {
        if (p) cudaFreeAsync(p, st);
    }
    cudaError_t alloc(size_t n) { return cudaMallocAsync(&p, sizeof(T) * (n ? n : 1), st); }
};

inline unsigned grid_for(int64_t n, int threads) {
    return (unsigned)((n + threads - 1) / threads);
}

// Sort the nodes by (pencil of W1 x W2 cells, lo0) into `ns` and cut the
// pencil runs into window tiles.
int order_and_tile(Plan &p, const double *a0, const double *a1, const double *a2, int W1, int W2,
                   const TileGeom &tg, NodeSet &ns, Tile **tiles, int64_t *ntiles, bool make_tiles,
                   cudaStream_t st, bool reuse_order = false) {
    const int64_t M = p.M;
    const int T = 256;
    if (!reuse_order) {
        SGL_CUDA_CHECK(cudaMalloc(&ns.u0, sizeof(double) * (M ? M : 1)));
        SGL_CUDA_CHECK(cudaMalloc(&ns.u1, sizeof(double) * (M ? M : 1)));
        SGL_CUDA_CHECK(cudaMalloc(&ns.u2, sizeof(double) * (M ? M : 1)));
        SGL_CUDA_CHECK(cudaMalloc(&ns.perm, sizeof(int32_t) * (M ? M : 1)));
    }
    ns.n = M;
    if (M == 0) return SGL_OK;
    KeyGeom kg{p.grid[0], p.grid[1], p.grid[2], W1, W2, (p.grid[2] + W2 - 1) / W2, 0, p.q};
    const uint64_t regular = (uint64_t)((p.grid[1] + W1 - 1) / W1) * kg.P2 * (uint64_t)p.grid[0];
    if (W1 > 1 || W2 > 1) kg.line_base = regular;
    DevBuf<uint64_t> key, key_s;
    DevBuf<int32_t> idx;
    SGL_CUDA_CHECK(key.alloc(M));
    SGL_CUDA_CHECK(key_s.alloc(M));
    SGL_CUDA_CHECK(idx.alloc(M));
    k_key<<<grid_for(M, T), T, 0, st>>>(a0, a1, a2, M, kg, key.p, idx.p);
    SGL_CUDA_CHECK(cudaGetLastError());
    // sort by (pencil, lo0); only the bits in use
    const uint64_t maxkey =
        regular + (kg.line_base ? (uint64_t)p.grid[1] * (uint64_t)p.grid[2] * (uint64_t)p.grid[0] : 0);
    int bits = 1;
    while (bits < 64 && (1ull << bits) < maxkey) ++bits;
    {
        DevBuf<int32_t> perm_tmp;
        if (reuse_order) SGL_CUDA_CHECK(perm_tmp.alloc(M));   // order already in ns; keys needed for the runs
        int32_t *perm_out = reuse_order ? perm_tmp.p : ns.perm;
        DevBuf<unsigned char> tmp;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_s.p, idx.p, perm_out, (int)M, 0, bits, st);
        SGL_CUDA_CHECK(tmp.alloc(tb));
        cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key_s.p, idx.p, perm_out, (int)M, 0, bits, st);
        SGL_CUDA_CHECK(cudaGetLastError());
    }
    if (!reuse_order) {
        k_permute<<<grid_for(M, T), T, 0, st>>>(ns.perm, M, a0, a1, a2, ns.u0, ns.u1, ns.u2);
        SGL_CUDA_CHECK(cudaGetLastError());
    }
    if (!make_tiles) return SGL_OK;

    // pencil runs
    DevBuf<int32_t> head, rank, starts, counts, offs;
    SGL_CUDA_CHECK(head.alloc(M));
    SGL_CUDA_CHECK(rank.alloc(M));
    k_run_heads<<<grid_for(M, T), T, 0, st>>>(key_s.p, M, (uint64_t)p.grid[0], head.p);
    {
        DevBuf<unsigned char> tmp;
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, head.p, rank.p, (int)M, st);
        SGL_CUDA_CHECK(tmp.alloc(tb));
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, head.p, rank.p, (int)M, st);
    }
    int32_t last_rank = 0, last_head = 0;
    SGL_CUDA_CHECK(cudaMemcpyAsync(&last_rank, rank.p + M - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaMemcpyAsync(&last_head, head.p + M - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    const int64_t nruns = (int64_t)last_rank + last_head;
    SGL_CUDA_CHECK(starts.alloc(nruns));
    SGL_CUDA_CHECK(counts.alloc(nruns));
    SGL_CUDA_CHECK(offs.alloc(nruns));
    k_run_starts<<<grid_for(M, T), T, 0, st>>>(head.p, rank.p, M, starts.p);
    k_tiles_warp<<<grid_for(nruns * 32, 256), 256, 0, st>>>(starts.p, nruns, M, ns.u0, ns.u1, ns.u2, tg, counts.p,
                                                           nullptr, nullptr);
    {
        DevBuf<unsigned char> tmp;
        size_t tb = 0;
        cub::DeviceScan::ExclusiveSum(nullptr, tb, counts.p, offs.p, (int)nruns, st);
        SGL_CUDA_CHECK(tmp.alloc(tb));
        cub::DeviceScan::ExclusiveSum(tmp.p, tb, counts.p, offs.p, (int)nruns, st);
    }
    int32_t lc = 0, lo = 0;
    SGL_CUDA_CHECK(cudaMemcpyAsync(&lc, counts.p + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaMemcpyAsync(&lo, offs.p + nruns - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    *ntiles = (int64_t)lc + lo;
    SGL_CUDA_CHECK(cudaMalloc(tiles, sizeof(Tile) * (*ntiles)));
    k_tiles_warp<<<grid_for(nruns * 32, 256), 256, 0, st>>>(starts.p, nruns, M, ns.u0, ns.u1, ns.u2, tg, counts.p,
                                                           offs.p, *tiles);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

__global__ void k_tile_band_key(const Tile *__restrict__ t, int64_t n, uint64_t *key, int32_t *idx) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    // box origins are >= -(pad + 8): bias them non-negative; 21 bits per field
    const uint64_t b0 = (uint64_t)((t[i].o0 >> 3) + 4096), b1 = (uint64_t)(t[i].o1 + 4096),
                   b2 = (uint64_t)(t[i].o2 + 4096);
    key[i] = (b0 << 42) | (b1 << 21) | b2;
    idx[i] = (int32_t)i;
}

__global__ void k_tile_gather(const Tile *__restrict__ src, const int32_t *__restrict__ idx, int64_t n,
                              Tile *__restrict__ dst) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) dst[i] = src[idx[i]];
}

// L2 order of a tile list (see build_nodes): a stable device radix sort by
// (axis-0 band of 8 slabs, o1, o2)
int reorder_tiles(Tile *tiles, int64_t n, cudaStream_t st) {
    if (n <= 1) return SGL_OK;
    DevBuf<uint64_t> key, key_s;
    DevBuf<int32_t> idx, idx_s;
    DevBuf<Tile> copy;
    SGL_CUDA_CHECK(key.alloc(n));
    SGL_CUDA_CHECK(key_s.alloc(n));
    SGL_CUDA_CHECK(idx.alloc(n));
    SGL_CUDA_CHECK(idx_s.alloc(n));
    SGL_CUDA_CHECK(copy.alloc(n));
    k_tile_band_key<<<grid_for(n, 256), 256, 0, st>>>(tiles, n, key.p, idx.p);
    SGL_CUDA_CHECK(cudaGetLastError());
    {
        DevBuf<unsigned char> tmp;
        size_t tb = 0;
        cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_s.p, idx.p, idx_s.p, (int)n, 0, 63, st);
        SGL_CUDA_CHECK(tmp.alloc(tb));
        cub::DeviceRadixSort::SortPairs(tmp.p, tb, key.p, key_s.p, idx.p, idx_s.p, (int)n, 0, 63, st);
        SGL_CUDA_CHECK(cudaGetLastError());
    }
    SGL_CUDA_CHECK(cudaMemcpyAsync(copy.p, tiles, sizeof(Tile) * n, cudaMemcpyDeviceToDevice, st));
    k_tile_gather<<<grid_for(n, 256), 256, 0, st>>>(copy.p, idx_s.p, n, tiles);
    SGL_CUDA_CHECK(cudaGetLastError());
    return SGL_OK;
}

// Work of an int8 tile in K-steps (as k_tile_stats counts it): mode 1 gather, mode 2 scatter
static inline int64_t i8_tile_work(const Tile &t, int mode) {
    if (mode == 1) return (i8::CHUNKS * t.e0 + 1) / 2;
    return (int64_t)((t.e0 * kI8Box2 + 127) / 128) * ((t.count + 31) / 32);
}

// Load balance of the persistent int8 window kernels: CTA c of G takes tiles
// c, c + G, c + 2G, ... of the (L2-ordered) list, so the per-CTA K-step sums
// differ by 1-2 % and the kernel ends with its slowest CTA.  The tiles are
// permuted within their rounds (the tiles that run at the same time stay the
// same: the L2 order is kept) so that, round by round from the last, the
// largest tile goes to the CTA with the smallest sum.  Host side, once per
// plan (tiles copied down and back).  Config 3: slowest CTA / mean K-steps
// 1.0235 -> 1.0082 with only the last eighth of the rounds permuted (scatter
// stage 28.46 -> 28.12 ms).
int balance_tiles(Tile *tiles, int64_t n, int mode, int G, cudaStream_t st, bool report) {
    if (G < 2 || n < 4 * (int64_t)G) return SGL_OK;
    const int64_t R = (n + G - 1) / G;                    // rounds (the last may be partial)
    const int64_t T = R;   // every round: tiles move within their round only
    const int64_t first = (R - T) * G;                    // first tile of the tail
    std::vector<Tile> h((size_t)n);
    SGL_CUDA_CHECK(cudaMemcpyAsync(h.data(), tiles, sizeof(Tile) * n, cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<int64_t> load((size_t)G, 0);
    for (int64_t i = 0; i < first; ++i) load[(size_t)(i % G)] += i8_tile_work(h[(size_t)i], mode);
    std::vector<Tile> out(h.begin() + first, h.end());
    std::vector<int> cta, tix;
    auto imbalance = [&](const std::vector<int64_t> &l) {   // slowest CTA over the mean
        int64_t mx = 0, sum = 0;
        for (int64_t v : l) mx = std::max(mx, v), sum += v;
        return sum > 0 ? (double)mx * G / (double)sum : 1.0;
    };
    double before = 1.0;
    if (report) {
        std::vector<int64_t> l0 = load;
        for (int64_t i = first; i < n; ++i) l0[(size_t)(i % G)] += i8_tile_work(h[(size_t)i], mode);
        before = imbalance(l0);
    }
    for (int64_t r = R - 1; r >= R - T; --r) {
        const int64_t b = r * G, e = std::min<int64_t>(n, b + G);
        const int k = (int)(e - b);                       // positions b + c, c < k, go to CTA c
        cta.resize((size_t)k);
        tix.resize((size_t)k);
        for (int c = 0; c < k; ++c) cta[(size_t)c] = tix[(size_t)c] = c;
        std::stable_sort(cta.begin(), cta.end(), [&](int x, int y) { return load[(size_t)x] < load[(size_t)y]; });
        std::stable_sort(tix.begin(), tix.end(), [&](int x, int y) {
            return i8_tile_work(h[(size_t)(b + x)], mode) > i8_tile_work(h[(size_t)(b + y)], mode);
        });
        for (int j = 0; j < k; ++j) {
            const Tile &t = h[(size_t)(b + tix[(size_t)j])];
            out[(size_t)(b - first + cta[(size_t)j])] = t;
            load[(size_t)cta[(size_t)j]] += i8_tile_work(t, mode);
        }
    }
    SGL_CUDA_CHECK(cudaMemcpyAsync(tiles + first, out.data(), sizeof(Tile) * (n - first), cudaMemcpyHostToDevice, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    if (report)
        fprintf(stderr, "int8 %s tiles: %lld over %d CTAs, slowest CTA / mean K-steps %.4f -> %.4f (%lld rounds)\n",
                mode == 1 ? "gather" : "scatter", (long long)n, G, before, imbalance(load), (long long)T);
    return SGL_OK;
}

// per-list tile statistics on the device (one pass, 64-bit atomics)
struct TileStatsDev {
    unsigned long long nodes, work, bad;
    int box;
};

__global__ void k_tile_stats(const Tile *__restrict__ tiles, int64_t n, int mode, WindowParams wp,
                             TileStatsDev *out) {
    unsigned long long nodes = 0, work = 0, bad = 0;
    int box = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const Tile t = tiles[i];
        nodes += (unsigned long long)t.count;
        if (mode == 0) {   // FP64 gather tiles: DMMA m8n8k4 of one pass, box limits
            const int64_t mt = (t.e1 + 3) / 4, ks = (t.e2 + 3) / 4, nt = (t.count + 7) / 8;
            work += (unsigned long long)(t.e0 * mt * ks * nt);
            box = max(box, max(t.e1, t.e2));
            bad |= (t.e1 > kBoxMax || t.e2 > kBoxMax || t.e0 > kBox0Max);
        } else {           // int8 tiles: K range of the digit boxes
            const int k0 = i8::kstart2(t, wp);
            bad |= (t.o2 + wp.pad < k0 || t.o2 + wp.pad + t.e2 > k0 + kI8Box2 || t.e1 > kI8Box1 ||
                    t.e0 > kBox0Max || t.count > (mode == 1 ? kI8Nodes : kI8SNodes));
            if (mode == 1) work += (unsigned long long)((i8::CHUNKS * t.e0 + 1) / 2);   // gather K-steps
            else work += (unsigned long long)(((t.e0 * kI8Box2 + 127) / 128) * ((t.count + 31) / 32));
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        nodes += __shfl_xor_sync(0xffffffffu, nodes, o);
        work += __shfl_xor_sync(0xffffffffu, work, o);
        bad |= __shfl_xor_sync(0xffffffffu, bad, o);
        box = max(box, __shfl_xor_sync(0xffffffffu, box, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&out->nodes, nodes);
        atomicAdd(&out->work, work);
        atomicOr(&out->bad, bad);
        atomicMax(&out->box, box);
    }
}

}  // namespace

int tile_stats(const Tile *tiles, int64_t n, int mode, const WindowParams &wp, cudaStream_t st, TileStats *out) {
    *out = TileStats();
    if (n <= 0) return SGL_OK;
    TileStatsDev *d = nullptr;
    SGL_CUDA_CHECK(cudaMallocAsync(&d, sizeof(TileStatsDev), st));
    SGL_CUDA_CHECK(cudaMemsetAsync(d, 0, sizeof(TileStatsDev), st));
    k_tile_stats<<<(unsigned)std::min<int64_t>(1024, (n + 255) / 256), 256, 0, st>>>(tiles, n, mode, wp, d);
    TileStatsDev h;
    SGL_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st));
    SGL_CUDA_CHECK(cudaFreeAsync(d, st));
    SGL_CUDA_CHECK(cudaStreamSynchronize(st));
    out->nodes = (int64_t)h.nodes;
    out->work = (int64_t)h.work;
    out->bad = h.bad != 0;
    out->box = h.box;
    return SGL_OK;
}

int resolve_rho(Plan &p, const double *pts, cudaStream_t st) {
    t_plan_stream = st;
    const int64_t M = p.M;
    const int T = 256;
    // rho: explicit, or the largest radius (choose_rho, transform.py:39-43)
    if (!p.raw && !(p.rho > 0)) {
        double rmax = 0.0;
        if (M > 0) {
            DevBuf<double> r, out;
            DevBuf<unsigned char> tmp;
            SGL_CUDA_CHECK(r.alloc(M));
            SGL_CUDA_CHECK(out.alloc(1));
            k_radius<<<grid_for(M, T), T, 0, st>>>(pts, M, r.p);
            size_t tb = 0;
            cub::DeviceReduce::Max(nullptr, tb, r.p, out.p, (int)M, st);
            SGL_CUDA_CHECK(tmp.alloc(tb));
            cub::DeviceReduce::Max(tmp.p, tb, r.p, out.p, (int)M, st);
            SGL_CUDA_CHECK(cudaMemcpyAsync(&rmax, out.p, sizeof(double), cudaMemcpyDeviceToHost, st));
            SGL_CUDA_CHECK(cudaStreamSynchronize(st));
        }
        p.rho = rmax > 0 ? rmax : 1.0;
    }
    if (M > 0 && !p.raw) {
        DevBuf<int> bad;
        SGL_CUDA_CHECK(bad.alloc(1));
        SGL_CUDA_CHECK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
        k_check_radius<<<grid_for(M, T), T, 0, st>>>(pts, M, p.rho * (1 + 1e-12), bad.p);
        int hb = 0;
        SGL_CUDA_CHECK(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        SGL_CUDA_CHECK(cudaStreamSynchronize(st));
        if (hb) {
            set_error("point radius exceeds the radial parameter rho");
            return SGL_EINVAL;
        }
    }
    return SGL_OK;
}

int build_nodes(Plan &p, const double *pts, cudaStream_t st) {
    t_plan_stream = st;
    const int64_t M = p.M;
    const int T = 256;
    DevBuf<double> a0, a1, a2;
    SGL_CUDA_CHECK(a0.alloc(M));
    SGL_CUDA_CHECK(a1.alloc(M));
    SGL_CUDA_CHECK(a2.alloc(M));
    if (M > 0) {
        if (p.raw)
            k_torus<<<grid_for(M, T), T, 0, st>>>(pts, M, p.d, p.grid[0], p.grid[1], p.grid[2], a0.p, a1.p, a2.p);
        else
            k_warp<<<grid_for(M, T), T, 0, st>>>(pts, M, p.rho, p.grid[0], p.grid[1], p.grid[2], a0.p, a1.p, a2.p);
        SGL_CUDA_CHECK(cudaGetLastError());
    }
    // Gather order: W x W pencils (cells on axes 1-2), nodes by lo0 inside a
    // pencil; 2q - 1 + W == 0 (mod 4) gives exact 4-row / 4-column DMMA tiles.
    // The wide cross-section keeps a 64-node tile within a few lo0 rows, so
    // the 8 consumer warps stay close together in the slab ring.
    int W = (4 - (2 * p.q - 1) % 4) % 4;
    if (W < 2) W += 4;
    plan_lap(p, st, "rho + warp");
    int rc = order_and_tile(p, a0.p, a1.p, a2.p, W, W, TileGeom{p.q, kBox0Max - 2 * p.q - 1, kTileNodes, kBox0Max},
                            p.nodes, &p.tiles, &p.n_tiles, !p.generic, st);
    plan_lap(p, st, "gather order + tiles");
    if (rc || p.generic) return rc;
    if (p.i8) {
        // int8 tensor-core gather: 8 x 16 pencils (box 40 x 48 = MMA N x 3 K-chunks per slab), 128-node tiles
        TileGeom ig{p.q, kBox0Max - 2 * p.q - 1, kI8Nodes, kBox0Max};
        ig.box1 = kI8Box1;
        ig.box2 = kI8Box2;
        rc = order_and_tile(p, a0.p, a1.p, a2.p, kI8Box1 - 32, kI8Box2 - 32, ig, p.inodes, &p.itiles, &p.n_itiles,
                            true, st);
        if (rc) return rc;
        plan_lap(p, st, "int8 order + tiles");
        rc = reorder_tiles(p.itiles, p.n_itiles, st);
        if (rc) return rc;
        rc = balance_tiles(p.itiles, p.n_itiles, 1, num_sms(), st, (p.flags & SGL_FLAG_I8_PROF) != 0);
        if (rc) return rc;
        plan_lap(p, st, "int8 tile reorder");
        if (p.i8s || p.i8s_auto) {
            // int8 scatter: same order, 512-node tiles (fewer grid REDs per node)
            TileGeom sg = ig;
            sg.max_nodes = kI8SNodes;
            rc = order_and_tile(p, a0.p, a1.p, a2.p, kI8Box1 - 32, kI8Box2 - 32, sg, p.inodes, &p.istiles,
                                &p.n_istiles, true, st, true);
            if (rc) return rc;
            rc = reorder_tiles(p.istiles, p.n_istiles, st);
            if (rc) return rc;
            rc = balance_tiles(p.istiles, p.n_istiles, 2, num_sms(), st, (p.flags & SGL_FLAG_I8_PROF) != 0);
            if (rc) return rc;
            if (!p.i8s) {
                // automatic choice: the int8 scatter beats the FP64 DMMA scatter on
                // every measured node set of >= 1.5e5 nodes up to 1.3 int8 K-steps
                // per node (config-3 subsamples, i.e. the node shards of a
                // strong-scaling run: 1.2-1.7x, profiles/r02/scatter_crossover.txt;
                // config 3: 29.7 vs 50 ms); below ~1e5 nodes its per-plan setup
                // (value-digit ring, guard calibration) is not worth it.  Inputs
                // the accuracy guard keeps rejecting switch the plan to FP64 at run
                // time (Plan::i8s_off, capi.cu)
                TileStats ts;
                rc = tile_stats(p.istiles, p.n_istiles, 2, p.wp, st, &ts);
                if (rc) return rc;
                const double ks = (double)ts.work;
                p.i8s = p.M >= 100000 && ks < 1.5 * (double)p.M;
                if (!p.i8s) {
                    cudaFree(p.istiles);
                    p.istiles = nullptr;
                    p.n_istiles = 0;
                }
            }
        }
    }
    // Scatter order: with dense nodes, W x W2 pencils whose axis-2 box is a
    // multiple of 8 (exact 8-column DMMA tiles, ~17 % fewer DMMAs; warps own
    // whole slabs, so a long lo0 span costs nothing); sparse node sets keep
    // the gather order, whose wider cross-section keeps enough nodes per tile
    // to amortise the RED of each box fragment.
    int W2 = (8 - (2 * p.q - 1) % 8) % 8;
    if (W2 < 1) W2 += 8;
    const double cells = (double)p.grid[0] * p.grid[1] * p.grid[2] / 4.0;   // nodes fill axes 0-1 up to pi
    const double per_row = (double)M / cells * W * W2;                        // nodes per lo0 row of a pencil
    bool narrow = W2 != W && per_row >= 1.5;   // crossover measured on the config-3 shape (r01)
    if (p.flags & SGL_FLAG_SCATTER_WIDE) narrow = false;   // experiments
    if (p.flags & SGL_FLAG_SCATTER_NARROW) narrow = W2 != W;
    plan_lap(p, st, "int8 scatter tiles");
    const TileGeom stg{p.q, kSBox0Max - 2 * p.q - 1, kSTileNodes, kSBox0Max};
    if (narrow) {
        rc = order_and_tile(p, a0.p, a1.p, a2.p, W, W2, stg, p.snodes, &p.stiles, &p.n_stiles, true, st);
    } else {
        p.snodes_shared = true;
        p.snodes = p.nodes;
        rc = order_and_tile(p, a0.p, a1.p, a2.p, W, W, stg, p.snodes, &p.stiles, &p.n_stiles, true, st, true);
    }
    if (rc) return rc;
    // L2 locality: CTAs walk the tile list with a grid stride, so the tiles in
    // flight at any moment are a contiguous stretch of the list.  Ordering the
    // list by axis-0 band first (then axis 1, axis 2) keeps that stretch inside
    // a narrow slab band of the grid instead of a few full-length pencils.
    plan_lap(p, st, "scatter order + tiles");
    rc = reorder_tiles(p.tiles, p.n_tiles, st);
    if (rc) return rc;
    rc = reorder_tiles(p.stiles, p.n_stiles, st);
    if (rc) return rc;
    plan_lap(p, st, "tile reorder");

    // tile statistics (device): nodes covered and DMMA count of one gather pass
    TileStats ts;
    rc = tile_stats(p.tiles, p.n_tiles, 0, p.wp, st, &ts);
    if (rc) return rc;
    if (ts.bad) {
        set_error("internal: window tile exceeds the box limits");
        return SGL_ECUDA;
    }
    p.tile_nodes = ts.nodes;
    p.tile_dmma = ts.work;
    p.tile_box = std::max(1, ts.box);
    return SGL_OK;
}

}  // namespace sgl
