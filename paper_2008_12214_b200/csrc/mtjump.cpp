// mtjump.cpp — jump-ahead for std::mt19937_64 (host side).
//
// The reference draws every random phase from one std::mt19937_64 stream
// (rng.hpp:23-67).  To generate a stream with many CTAs at once, each CTA must
// start at a known draw offset J.  The engine is F2-linear: with W_n the
// window (x_n .. x_{n+311}) of raw words and P(x) the characteristic
// polynomial of the transition (degree 19937), W_{1+J} = g(F) W_1 for
// g = x^J mod P, i.e. window word j of W_{1+J} is XOR_{i : g_i = 1} x_{1+i+j}.
// (W_1 rather than W_0: the 31 low bits of x_0 are dead state, annihilated
// after one step.)  This file computes P (Berlekamp-Massey on one output bit)
// and g for a given J; the device applies g (mt64.cuh, k_mt_jump).
#if defined(__PCLMUL__)
#include <wmmintrin.h>
#endif

#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "mtjump.h"

namespace hg {
namespace {

constexpr int kN = 312, kM = 156;
constexpr uint64_t kUM = 0xFFFFFFFF80000000ull, kLM = 0x7FFFFFFFull, kA = 0xB5026F5AA96619E9ull;

struct HostMt {  // std::mt19937_64 raw-word generator (untempered words x_0, x_1, ...)
    std::vector<uint64_t> x;
    explicit HostMt(uint64_t seed) {
        x.resize(kN);
        x[0] = seed;
        for (int i = 1; i < kN; ++i) x[i] = 6364136223846793005ull * (x[i - 1] ^ (x[i - 1] >> 62)) + (uint64_t)i;
    }
    uint64_t word(size_t n) {  // x_n, extending the sequence with x_{n+312} = x_{n+156} ^ mix(x_n, x_{n+1})
        while (x.size() <= n) {
            size_t k = x.size() - kN;
            uint64_t y = (x[k] & kUM) | (x[k + 1] & kLM);
            x.push_back(x[k + kM] ^ (y >> 1) ^ ((y & 1) ? kA : 0));
        }
        return x[n];
    }
};

using Poly = std::vector<uint64_t>;  // GF(2)[x], bit i of word i/64 = coefficient of x^i

inline int deg(const Poly& p) {
    for (int w = (int)p.size() - 1; w >= 0; --w)
        if (p[w]) return w * 64 + 63 - __builtin_clzll(p[w]);
    return -1;
}
inline bool bit(const Poly& p, int i) { return (p[i >> 6] >> (i & 63)) & 1; }
inline void setbit(Poly& p, int i) { p[i >> 6] ^= 1ull << (i & 63); }

// Berlekamp-Massey over GF(2): minimal connection polynomial of s (one byte
// per coefficient so the inner loops vectorise).
Poly berlekamp_massey(const std::vector<uint8_t>& s) {
    const int n = (int)s.size();
    std::vector<uint8_t> C(n + 1, 0), B(n + 1, 0), T;
    C[0] = B[0] = 1;
    int L = 0, m = 1;
    for (int i = 0; i < n; ++i) {
        uint8_t d = s[i];
        const uint8_t* si = s.data() + i;
        for (int j = 1; j <= L; ++j) d ^= C[j] & si[-j];
        if (!d) {
            ++m;
            continue;
        }
        const bool grow = 2 * L <= i;
        if (grow) T = C;
        for (int j = 0; j + m <= n; ++j) C[j + m] ^= B[j];
        if (grow) {
            L = i + 1 - L;
            B.swap(T);
            m = 1;
        } else {
            ++m;
        }
    }
    Poly out(L / 64 + 1, 0);
    for (int j = 0; j <= L; ++j)
        if (C[j]) setbit(out, j);
    return out;
}

struct Field {
    int L = 0;                 // degree of P (19937)
    int W = 0;                 // words of a reduced polynomial
    Poly P;                    // characteristic polynomial
    std::vector<Poly> table;   // table[b] = (b * x^L) mod P for 8-bit b (b placed at bits L..L+7)

    Field() {
        // output bit 0 of the raw words x_{312+n}: a linear function of the state
        HostMt g(5489);
        const int n = 2 * 19937 + 64;
        std::vector<uint8_t> s(n);
        for (int i = 0; i < n; ++i) s[i] = (uint8_t)(g.word(kN + i) & 1);
        Poly C = berlekamp_massey(s);
        L = deg(C);
        // characteristic polynomial P(x) = x^L C(1/x)
        W = L / 64 + 1;
        P.assign(W + 1, 0);
        for (int i = 0; i <= L; ++i)
            if (bit(C, i)) setbit(P, L - i);
        // reduction table: for each byte value b, (b(x) * x^L) mod P
        table.resize(256);
        std::vector<Poly> xk(8);  // x^(L+k) mod P, k = 0..7
        Poly cur(W + 1, 0);
        for (int i = 0; i < L; ++i)  // x^L = P - x^L (mod P) = low part of P
            if (bit(P, i)) setbit(cur, i);
        for (int k = 0; k < 8; ++k) {
            xk[k] = cur;
            // cur *= x (mod P)
            const bool top = bit(cur, L - 1);
            for (int w = W; w > 0; --w) cur[w] = (cur[w] << 1) | (cur[w - 1] >> 63);
            cur[0] <<= 1;
            if (top) {
                setbit(cur, L);  // clear x^L, add low part of P
                for (int i = 0; i < L; ++i)
                    if (bit(P, i)) setbit(cur, i);
            }
        }
        for (int b = 0; b < 256; ++b) {
            Poly t(W + 1, 0);
            for (int k = 0; k < 8; ++k)
                if ((b >> k) & 1)
                    for (int w = 0; w <= W; ++w) t[w] ^= xk[k][w];
            table[b] = t;
        }
    }

    // a (degree < 2L) mod P: windows of 8 coefficients at positions L+8k .. L+8k+7,
    // from the top down, each replaced by table[b] * x^(8k) (degree < L+8k).
    Poly reduce(Poly a) const {
        const int need = (2 * L + 16) / 64 + 2;
        if ((int)a.size() < need) a.resize(need, 0);
        for (int k = (2 * L - L) / 8 + 1; k >= 0; --k) {
            const int t = L + 8 * k;
            const int w = t >> 6, o = t & 63;
            uint32_t b = (uint32_t)(a[w] >> o);
            if (o > 56) b |= (uint32_t)(a[w + 1] << (64 - o));
            b &= 255;
            if (!b) continue;
            // clear the window
            a[w] &= ~(255ull << o);
            if (o > 56) a[w + 1] &= ~(255ull >> (64 - o));
            // add table[b] << 8k
            const Poly& e = table[b];
            const int s = 8 * k, sw = s >> 6, sb = s & 63;
            if (sb == 0) {
                for (int i = 0; i <= W; ++i) a[i + sw] ^= e[i];
            } else {
                for (int i = 0; i <= W; ++i) {
                    a[i + sw] ^= e[i] << sb;
                    a[i + sw + 1] ^= e[i] >> (64 - sb);
                }
            }
        }
        a.resize(W);
        return a;
    }

    // carry-less product (PCLMULQDQ when built with -mpclmul), then reduction
    static inline void clmul64(uint64_t a, uint64_t b, uint64_t& lo, uint64_t& hi) {
#if defined(__PCLMUL__)
        const __m128i p = _mm_clmulepi64_si128(_mm_set_epi64x(0, (long long)a), _mm_set_epi64x(0, (long long)b), 0x00);
        lo = (uint64_t)_mm_cvtsi128_si64(p);
        hi = (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(p, p));
#else
        lo = hi = 0;
        for (int k = 0; k < 64; ++k)
            if ((b >> k) & 1) {
                lo ^= a << k;
                if (k) hi ^= a >> (64 - k);
            }
#endif
    }
    Poly mulmod(const Poly& a, const Poly& b) const {
        Poly r(2 * W + 2, 0);
        for (int i = 0; i < W; ++i) {
            if (!a[i]) continue;
            for (int j = 0; j < W; ++j) {
                if (!b[j]) continue;
                uint64_t lo, hi;
                clmul64(a[i], b[j], lo, hi);
                r[i + j] ^= lo;
                r[i + j + 1] ^= hi;
            }
        }
        return reduce(r);
    }
};

const Field& field() {
    static Field f;
    return f;
}

}  // namespace

int mt_charpoly_degree() { return field().L; }

// g = x^J mod P (J >= 0), as kMtPolyWords words.
void mt_jump_poly(uint64_t J, uint64_t* out) {
    static std::mutex mu;
    static std::map<uint64_t, Poly> cache;
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(J);
        if (it != cache.end()) {
            std::memcpy(out, it->second.data(), sizeof(uint64_t) * kMtPolyWords);
            return;
        }
    }
    const Field& F = field();
    Poly g(F.W, 0);
    g[0] = 1;
    Poly x(F.W, 0);
    x[0] = 2;
    // left-to-right binary exponentiation
    int top = 63;
    while (top >= 0 && !((J >> top) & 1)) --top;
    for (int b = top; b >= 0; --b) {
        g = F.mulmod(g, g);
        if ((J >> b) & 1) g = F.mulmod(g, x);
    }
    g.resize(kMtPolyWords, 0);
    std::lock_guard<std::mutex> lk(mu);
    cache[J] = g;
    std::memcpy(out, g.data(), sizeof(uint64_t) * kMtPolyWords);
}

const std::vector<uint64_t>& mt_chunk_polys(uint64_t offset0, uint64_t len, int chunks) {
    static std::mutex mu;
    static std::map<std::tuple<uint64_t, uint64_t, int>, std::vector<uint64_t>> cache;
    const auto key = std::make_tuple(offset0, len, chunks);
    {
        std::lock_guard<std::mutex> lk(mu);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
    }
    const Field& F = field();
    const int c_first = offset0 == 0 ? 1 : 0;
    std::vector<uint64_t> out;
    if (chunks > c_first) {
        out.assign((size_t)(chunks - c_first) * kMtPolyWords, 0);
        Poly cur(kMtPolyWords), step(kMtPolyWords);
        mt_jump_poly(offset0 + (uint64_t)c_first * len - 1, cur.data());
        mt_jump_poly(len, step.data());
        cur.resize(F.W);
        step.resize(F.W);
        for (int c = c_first; c < chunks; ++c) {
            if (c > c_first) cur = F.mulmod(cur, step);
            std::memcpy(out.data() + (size_t)(c - c_first) * kMtPolyWords, cur.data(), sizeof(uint64_t) * F.W);
        }
    }
    std::lock_guard<std::mutex> lk(mu);
    return cache.emplace(key, std::move(out)).first->second;
}

void mt_poly_offsets(const uint64_t* polys, int npolys, std::vector<int>& starts, std::vector<uint16_t>& pool) {
    constexpr int kBlocks = (kMtPolyWords * 64 + kN - 1) / kN;  // 64
    starts.assign((size_t)npolys * (kBlocks + 1), 0);
    pool.clear();
    for (int k = 0; k < npolys; ++k) {
        const uint64_t* g = polys + (size_t)k * kMtPolyWords;
        for (int q = 0; q < kBlocks; ++q) {
            starts[(size_t)k * (kBlocks + 1) + q] = (int)pool.size();
            for (int ii = 0; ii < kN; ++ii) {
                const int i = q * kN + ii;
                if (i < kMtPolyWords * 64 && ((g[i >> 6] >> (i & 63)) & 1)) pool.push_back((uint16_t)ii);
            }
        }
        starts[(size_t)k * (kBlocks + 1) + kBlocks] = (int)pool.size();
    }
}

// Host reference of the jump: the raw-word window after J draws of the engine
// seeded with `engine_seed` (words x_J .. x_{J+311}), computed as g(F) W_1.
void mt_jump_state_host(uint64_t engine_seed, uint64_t J, uint64_t* window) {
    if (J == 0) {
        HostMt m(engine_seed);
        for (int j = 0; j < kN; ++j) window[j] = m.word(j);
        return;
    }
    std::vector<uint64_t> g(kMtPolyWords);
    mt_jump_poly(J - 1, g.data());
    HostMt m(engine_seed);
    std::vector<uint64_t> acc(kN, 0);
    for (int i = 0; i < kMtPolyWords * 64; ++i)
        if ((g[i >> 6] >> (i & 63)) & 1)
            for (int j = 0; j < kN; ++j) acc[j] ^= m.word(1 + (size_t)i + j);
    std::memcpy(window, acc.data(), sizeof(uint64_t) * kN);
}

}  // namespace hg
