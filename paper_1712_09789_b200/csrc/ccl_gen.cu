// ccl_gen.cu — random_image on the GPU, byte-identical
// with the reference generator (/root/reference/proj/src/generate.cpp:9-18,
// generate.hpp:15-43): pixel p is 1 iff (x_p >> 11) < density * 2^53, where
// x_p is the p-th xoshiro256** output after splitmix64 seeding.
//
// xoshiro256's state update is linear over GF(2): s_{n+1} = T s_n.  With p(x)
// the characteristic polynomial of T (Berlekamp-Massey on one state bit, once
// per process), jumping n steps is s_n = q(T) s_0 where q = x^n mod p: apply q
// by stepping the generator 256 times and XOR-accumulating the states at the
// set coefficients.  Each thread generates a chunk of CH consecutive pixels;
// its start is reached with two jumps (block start, then thread offset) whose
// polynomials come from host tables.
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <vector>

#include "ccl_internal.h"

namespace cclk {

namespace {

constexpr int GEN_THREADS = 256;
constexpr uint32_t GEN_CH = 2048;  // pixels per thread (multiple of 16)

struct P256 {
    uint64_t w[4];
};

// ---------------------------------------------------------------- host GF(2)[x]
inline bool bit(const P256& a, int i) { return (a.w[i >> 6] >> (i & 63)) & 1u; }

struct Charpoly {
    P256 low;  // p(x) = x^256 + low(x)
};

// Minimal polynomial of one output bit sequence of the linear state (bit 0 of
// s[0]) by Berlekamp-Massey over GF(2); degree 256 for xoshiro256.
Charpoly charpoly() {
    uint64_t s[4] = {0x9e3779b97f4a7c15ull, 0xbf58476d1ce4e5b9ull, 0x94d049bb133111ebull, 1ull};
    std::vector<int> seq(512);
    for (int n = 0; n < 512; ++n) {
        seq[n] = int(s[0] & 1u);
        const uint64_t t = s[1] << 17;
        s[2] ^= s[0];
        s[3] ^= s[1];
        s[1] ^= s[2];
        s[0] ^= s[3];
        s[2] ^= t;
        s[3] = (s[3] << 45) | (s[3] >> 19);
    }
    std::vector<int> c(513, 0), b(513, 0);
    c[0] = b[0] = 1;
    int L = 0, m = -1;
    for (int n = 0; n < 512; ++n) {
        int d = seq[n];
        for (int i = 1; i <= L; ++i) d ^= c[i] & seq[n - i];
        if (!d) continue;
        std::vector<int> t = c;
        for (int i = 0; i + n - m <= 512; ++i) c[i + n - m] ^= b[i];
        if (2 * L <= n) {
            L = n + 1 - L;
            m = n;
            b = t;
        }
    }
    // connection polynomial C(x) = 1 + c1 x + ... + cL x^L; characteristic
    // polynomial = x^L C(1/x) = x^L + c1 x^{L-1} + ... + cL
    Charpoly cp{};
    for (int i = 1; i <= L; ++i)
        if (c[i]) cp.low.w[(L - i) >> 6] |= 1ull << ((L - i) & 63);
    return cp;
}

// a * x mod p
inline P256 mulx(P256 a, const Charpoly& cp) {
    const bool top = (a.w[3] >> 63) & 1u;
    for (int i = 3; i > 0; --i) a.w[i] = (a.w[i] << 1) | (a.w[i - 1] >> 63);
    a.w[0] <<= 1;
    if (top)
        for (int i = 0; i < 4; ++i) a.w[i] ^= cp.low.w[i];
    return a;
}
// a * b mod p (Horner over the bits of b)
P256 mulmod(const P256& a, const P256& b, const Charpoly& cp) {
    P256 r{};
    for (int i = 255; i >= 0; --i) {
        r = mulx(r, cp);
        if (bit(b, i))
            for (int k = 0; k < 4; ++k) r.w[k] ^= a.w[k];
    }
    return r;
}
// x^n mod p
P256 xpow(uint64_t n, const Charpoly& cp) {
    P256 r{}, base{};
    r.w[0] = 1;
    base.w[0] = 2;  // x
    while (n) {
        if (n & 1u) r = mulmod(r, base, cp);
        base = mulmod(base, base, cp);
        n >>= 1;
    }
    return r;
}

const Charpoly& cached_charpoly() {
    static std::once_flag once;
    static Charpoly cp;
    std::call_once(once, [] { cp = charpoly(); });
    return cp;
}

// ---------------------------------------------------------------- device
__device__ __forceinline__ uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
__device__ __forceinline__ void step(uint64_t s[4]) {
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
}
__device__ __forceinline__ void jump(uint64_t s[4], const P256& q) {
    uint64_t a[4] = {0, 0, 0, 0};
    for (int i = 0; i < 256; ++i) {
        if ((q.w[i >> 6] >> (i & 63)) & 1u) {
            a[0] ^= s[0];
            a[1] ^= s[1];
            a[2] ^= s[2];
            a[3] ^= s[3];
        }
        step(s);
    }
    s[0] = a[0];
    s[1] = a[1];
    s[2] = a[2];
    s[3] = a[3];
}

__global__ void __launch_bounds__(GEN_THREADS) k_gen_random(uint8_t* out, uint64_t n, uint64_t thr, uint4 s01, uint4 s23,
                                                            const P256* block_jump, const P256* thread_jump) {
    const uint64_t first = (uint64_t(blockIdx.x) * GEN_THREADS + threadIdx.x) * GEN_CH;
    if (first >= n) return;
    uint64_t s[4] = {uint64_t(s01.x) | uint64_t(s01.y) << 32, uint64_t(s01.z) | uint64_t(s01.w) << 32,
                     uint64_t(s23.x) | uint64_t(s23.y) << 32, uint64_t(s23.z) | uint64_t(s23.w) << 32};
    jump(s, block_jump[blockIdx.x]);
    jump(s, thread_jump[threadIdx.x]);
    const uint64_t cnt = min(uint64_t(GEN_CH), n - first);
    uint8_t* dst = out + first;
    for (uint64_t i = 0; i < cnt; i += 16) {
        uint32_t wds[4] = {0, 0, 0, 0};
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const uint64_t x = rotl(s[1] * 5, 7) * 9;  // xoshiro256** output
            step(s);
            wds[k >> 2] |= uint32_t((x >> 11) < thr) << (8 * (k & 3));
        }
        if (i + 16 <= cnt) {
            *reinterpret_cast<uint4*>(dst + i) = make_uint4(wds[0], wds[1], wds[2], wds[3]);
        } else {
            for (uint64_t k = 0; i + k < cnt; ++k) dst[i + k] = uint8_t(wds[k >> 2] >> (8 * (k & 3)));
        }
    }
}

}  // namespace

// out: n bytes, contiguous, 16-byte aligned = pixels [first, first + n) of the
// image's raster stream (a strip of rows when first = row0 * w).
cudaError_t launch_gen_random(uint8_t* out, uint64_t n, uint64_t first, double density, uint64_t seed,
                              cudaStream_t s) {
    const Charpoly& cp = cached_charpoly();
    // splitmix64 seeding (generate.hpp:17-26)
    uint64_t st[4], x = seed;
    for (int i = 0; i < 4; ++i) {
        x += 0x9e3779b97f4a7c15ull;
        uint64_t z = x;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        st[i] = z ^ (z >> 31);
    }
    const uint64_t per_block = uint64_t(GEN_THREADS) * GEN_CH;
    const uint64_t nblocks = (n + per_block - 1) / per_block;
    std::vector<P256> tab(nblocks + GEN_THREADS);
    {   // block starts b * per_block, thread offsets t * GEN_CH: iterated products
        static std::once_flag once;
        static P256 xb, xc;
        std::call_once(once, [&] {
            xb = xpow(per_block, cp);
            xc = xpow(GEN_CH, cp);
        });
        P256 one{};
        one.w[0] = 1;
        P256 acc = first ? xpow(first, cp) : one;
        for (uint64_t b = 0; b < nblocks; ++b) {
            tab[b] = acc;
            acc = mulmod(acc, xb, cp);
        }
        acc = one;
        for (int t = 0; t < GEN_THREADS; ++t) {
            tab[nblocks + t] = acc;
            acc = mulmod(acc, xc, cp);
        }
    }
    P256* d_tab = nullptr;
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&d_tab), tab.size() * sizeof(P256), s);
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(d_tab, tab.data(), tab.size() * sizeof(P256), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) {
        const uint64_t thr = uint64_t(density * 9007199254740992.0);  // density * 2^53 (generate.cpp:13)
        const uint4 s01 = make_uint4(uint32_t(st[0]), uint32_t(st[0] >> 32), uint32_t(st[1]), uint32_t(st[1] >> 32));
        const uint4 s23 = make_uint4(uint32_t(st[2]), uint32_t(st[2] >> 32), uint32_t(st[3]), uint32_t(st[3] >> 32));
        k_gen_random<<<unsigned(nblocks), GEN_THREADS, 0, s>>>(out, n, thr, s01, s23, d_tab, d_tab + nblocks);
        e = cudaGetLastError();
        // the pageable source of the async copy must outlive it
        const cudaError_t e2 = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = e2;
    }
    const cudaError_t e3 = cudaFreeAsync(d_tab, s);
    return e != cudaSuccess ? e : e3;
}

}  // namespace cclk
