// model_digest on the host, natively: canonical json-curves serialization of
// a packed model, byte-identical to
//   json.dumps(model_to_dict(model), sort_keys=True, separators=(",", ":"))
// (linkcert/model_io.py:122-172), and its SHA-256 — the digest computed by
// compute_linking_matrix and verify (certify.py:163,188).
//
// Floats follow CPython's float.__repr__: shortest round-trip digits
// (Dragonbox via fmt, checked against std::to_chars), fixed notation when -4 < decpt <= 16 with ".0" for
// integral values, otherwise d[.ddd]e(+|-)XX with at least two exponent
// digits.  Formatting runs on worker threads chunk by chunk while the calling
// thread streams finished chunks, in order, through SHA-256 (SHA-NI when the
// CPU has it), so the digest costs ~max(format / threads, hash).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <charconv>
#include <cmath>
#include <condition_variable>
#include <cpuid.h>
#include <cstdint>
#include <cstring>
#include <immintrin.h>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#define FMT_HEADER_ONLY
#include <fmt/format.h>

#include "../../include/linkcert_b200.h"

namespace {

// ------------------------------------------------------------ float repr

// Layout of a shortest digit string d1 d2 ... dnd x 10^(exp10 - nd + 1) in
// float.__repr__ style (Objects/floatobject.c float_repr -> 'r' format).
char *put_digits(char *p, const char *digits, int nd, int exp10) {
    const int decpt = exp10 + 1;
    if (decpt <= -4 || decpt > 16) {
        *p++ = digits[0];
        if (nd > 1) {
            *p++ = '.';
            std::memcpy(p, digits + 1, nd - 1);
            p += nd - 1;
        }
        *p++ = 'e';
        *p++ = exp10 < 0 ? '-' : '+';
        int a = exp10 < 0 ? -exp10 : exp10;
        if (a >= 100) {
            *p++ = char('0' + a / 100);
            a %= 100;
        }
        *p++ = char('0' + a / 10);
        *p++ = char('0' + a % 10);
    } else if (decpt <= 0) {
        *p++ = '0';
        *p++ = '.';
        for (int k = 0; k < -decpt; ++k) *p++ = '0';
        std::memcpy(p, digits, nd);
        p += nd;
    } else if (decpt >= nd) {
        std::memcpy(p, digits, nd);
        p += nd;
        for (int k = nd; k < decpt; ++k) *p++ = '0';
        *p++ = '.';
        *p++ = '0';
    } else {
        std::memcpy(p, digits, decpt);
        p += decpt;
        *p++ = '.';
        std::memcpy(p, digits + decpt, nd - decpt);
        p += nd - decpt;
    }
    return p;
}

// Non-finite values and the cross-check path: std::to_chars (Ryu) shortest
// scientific digits, re-laid out.
char *put_repr_tochars(char *p, double x) {
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof buf, x, std::chars_format::scientific);
    const char *b = buf, *e = r.ptr;
    if (*b == '-') *p++ = *b++;
    if (!std::isfinite(x)) {
        std::memcpy(p, b, (size_t)(e - b));
        return p + (e - b);
    }
    char digits[32];
    int nd = 0;
    const char *q = b;
    for (; q < e && *q != 'e'; ++q)
        if (*q != '.') digits[nd++] = *q;
    int exp10 = 0;
    if (q < e) {
        ++q;
        const bool neg = *q == '-';
        if (*q == '+' || *q == '-') ++q;
        for (; q < e; ++q) exp10 = exp10 * 10 + (*q - '0');
        if (neg) exp10 = -exp10;
    }
    while (nd > 1 && digits[nd - 1] == '0') --nd;
    return put_digits(p, digits, nd, exp10);
}

const char kPairs[201] =
    "0001020304050607080910111213141516171819202122232425262728293031323334353637383940414243444546474849"
    "5051525354555657585960616263646566676869707172737475767778798081828384858687888990919293949596979899";

inline void put8(char *out, uint32_t v) {   // exactly 8 digits, leading zeros kept
    const uint32_t hi = v / 10000, lo = v % 10000;
    std::memcpy(out, kPairs + 2 * (hi / 100), 2);
    std::memcpy(out + 2, kPairs + 2 * (hi % 100), 2);
    std::memcpy(out + 4, kPairs + 2 * (lo / 100), 2);
    std::memcpy(out + 6, kPairs + 2 * (lo % 100), 2);
}

constexpr uint64_t kPow10[20] = {1ull,
                                 10ull,
                                 100ull,
                                 1000ull,
                                 10000ull,
                                 100000ull,
                                 1000000ull,
                                 10000000ull,
                                 100000000ull,
                                 1000000000ull,
                                 10000000000ull,
                                 100000000000ull,
                                 1000000000000ull,
                                 10000000000000ull,
                                 100000000000000ull,
                                 1000000000000000ull,
                                 10000000000000000ull,
                                 100000000000000000ull,
                                 1000000000000000000ull,
                                 10000000000000000000ull};

// Decimal digits of 1 <= n < 10^17 (a double's shortest significand), most
// significant first, via independent 8-digit halves; returns the count.
inline int u64_digits(uint64_t n, char *out) {
    const int bits = 64 - __builtin_clzll(n);
    int nd = (bits * 1233) >> 12;          // floor(log10(2^bits)) approximation
    nd += n >= kPow10[nd];
    char buf[40];
    const uint64_t top = n / 10000000000000000ull;   // digit 17 (0 or 1..9)
    const uint64_t rest = n % 10000000000000000ull;
    buf[0] = char('0' + top);
    put8(buf + 1, (uint32_t)(rest / 100000000u));
    put8(buf + 9, (uint32_t)(rest % 100000000u));
    std::memcpy(out, buf + 17 - nd, 17);   // out has >= 17 bytes
    return nd;
}

// float.__repr__: the shortest digit string that rounds back to x, the one
// closest to x among those (David Gay's mode 0, which CPython uses).  The
// shortest-closest decimal comes from fmt's Dragonbox (header-only, PyTorch's
// vendored fmt), which implements exactly that selection.
char *put_repr(char *p, double x) {
    if (!std::isfinite(x)) return put_repr_tochars(p, x);
    if (std::signbit(x)) *p++ = '-';
    if (x == 0.0) {
        std::memcpy(p, "0.0", 3);
        return p + 3;
    }
    const auto d = fmt::detail::dragonbox::to_decimal(std::fabs(x));
    char digits[24];
    int nd = u64_digits(d.significand, digits);
    int exp10 = d.exponent + nd - 1;
    while (nd > 1 && digits[nd - 1] == '0') --nd;
    return put_digits(p, digits, nd, exp10);
}

inline char *put(char *p, const char *s) {
    const size_t n = std::strlen(s);
    std::memcpy(p, s, n);
    return p + n;
}

char *put_triple(char *p, const double *v) {
    *p++ = '[';
    p = put_repr(p, v[0]);
    *p++ = ',';
    p = put_repr(p, v[1]);
    *p++ = ',';
    p = put_repr(p, v[2]);
    *p++ = ']';
    return p;
}

constexpr size_t kReprMax = 24;   // "-1.2345678901234567e-308"
constexpr size_t kTripleMax = 3 * kReprMax + 4;

// model_io.py:126: polyline iff a2 = a3 = 0 everywhere and every domain is [0, 1].
bool loop_is_polyline(const double *coeffs, const double *t, int64_t m) {
    for (int64_t k = 0; k < m; ++k) {
        const double *c = coeffs + 12 * k;
        for (int d = 6; d < 12; ++d)
            if (c[d] != 0.0) return false;
        if (t[2 * k] != 0.0 || t[2 * k + 1] != 1.0) return false;
    }
    return true;
}

size_t loop_bound(int64_t m, bool poly) {
    return 64 + (size_t)(m + 1) * (poly ? kTripleMax + 1 : 4 * kTripleMax + 2 * kReprMax + 24);
}

// One loop dict with sorted keys (model_io.py:124-145).
char *put_loop(char *p, const double *coeffs, const double *t, int64_t m, bool closed, bool poly) {
    p = put(p, closed ? "{\"closed\":true," : "{\"closed\":false,");
    if (poly) {
        p = put(p, "\"points\":[");
        for (int64_t k = 0; k < m; ++k) {
            if (k) *p++ = ',';
            p = put_triple(p, coeffs + 12 * k);
        }
        if (!closed && m > 0) {
            // loop.end_points()[-1]: eval_cubics at t = 1 (geometry.py:110)
            const double *c = coeffs + 12 * (m - 1);
            double e[3];
            for (int d = 0; d < 3; ++d) e[d] = ((c[d] + c[3 + d] * 1.0) + (c[6 + d] * 1.0) * 1.0) + c[9 + d] * 1.0;
            *p++ = ',';
            p = put_triple(p, e);
        }
        p = put(p, "],\"type\":\"polyline\"}");
    } else {
        p = put(p, "\"segments\":[");
        for (int64_t k = 0; k < m; ++k) {
            if (k) *p++ = ',';
            p = put(p, "{\"coeffs\":[");
            for (int r = 0; r < 4; ++r) {
                if (r) *p++ = ',';
                p = put_triple(p, coeffs + 12 * k + 3 * r);
            }
            p = put(p, "],\"t\":[");
            p = put_repr(p, t[2 * k]);
            *p++ = ',';
            p = put_repr(p, t[2 * k + 1]);
            p = put(p, "]}");
        }
        p = put(p, "],\"type\":\"cubics\"}");
    }
    return p;
}

// A closed from_polyline loop given by its vertex rows (n, 3): the "points" of
// model_to_dict are coeffs[:, 0] = the vertices (model_io.py:126-133).
char *put_loop_vertices(char *p, const double *v, int64_t m) {
    p = put(p, "{\"closed\":true,\"points\":[");
    for (int64_t k = 0; k < m; ++k) {
        if (k) *p++ = ',';
        p = put_triple(p, v + 3 * k);
    }
    return put(p, "],\"type\":\"polyline\"}");
}

// --------------------------------------------------------------- SHA-256

const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

inline uint32_t ror(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void sha256_blocks_portable(uint32_t s[8], const uint8_t *data, size_t nblocks) {
    for (; nblocks; --nblocks, data += 64) {
        uint32_t w[64];
        for (int i = 0; i < 16; ++i)
            w[i] = (uint32_t)data[4 * i] << 24 | (uint32_t)data[4 * i + 1] << 16 | (uint32_t)data[4 * i + 2] << 8 |
                   (uint32_t)data[4 * i + 3];
        for (int i = 16; i < 64; ++i) {
            const uint32_t s0 = ror(w[i - 15], 7) ^ ror(w[i - 15], 18) ^ (w[i - 15] >> 3);
            const uint32_t s1 = ror(w[i - 2], 17) ^ ror(w[i - 2], 19) ^ (w[i - 2] >> 10);
            w[i] = w[i - 16] + s0 + w[i - 7] + s1;
        }
        uint32_t a = s[0], b = s[1], c = s[2], d = s[3], e = s[4], f = s[5], g = s[6], h = s[7];
        for (int i = 0; i < 64; ++i) {
            const uint32_t S1 = ror(e, 6) ^ ror(e, 11) ^ ror(e, 25);
            const uint32_t ch = (e & f) ^ (~e & g);
            const uint32_t t1 = h + S1 + ch + K256[i] + w[i];
            const uint32_t S0 = ror(a, 2) ^ ror(a, 13) ^ ror(a, 22);
            const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
            const uint32_t t2 = S0 + mj;
            h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
        }
        s[0] += a; s[1] += b; s[2] += c; s[3] += d; s[4] += e; s[5] += f; s[6] += g; s[7] += h;
    }
}

__attribute__((target("sha,sse4.1,ssse3")))
void sha256_blocks_shani(uint32_t s[8], const uint8_t *data, size_t nblocks) {
    const __m128i MASK = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
    __m128i tmp = _mm_loadu_si128((const __m128i *)&s[0]);
    __m128i st1 = _mm_loadu_si128((const __m128i *)&s[4]);
    tmp = _mm_shuffle_epi32(tmp, 0xB1);            // CDAB
    st1 = _mm_shuffle_epi32(st1, 0x1B);            // EFGH
    __m128i st0 = _mm_alignr_epi8(tmp, st1, 8);    // ABEF
    st1 = _mm_blend_epi16(st1, tmp, 0xF0);         // CDGH
    for (; nblocks; --nblocks, data += 64) {
        const __m128i abef = st0, cdgh = st1;
        __m128i w0, w1, w2, w3;
#define SHA_ROUNDS(X, I)                                                                     \
    {                                                                                        \
        __m128i msg = _mm_add_epi32(X, _mm_loadu_si128((const __m128i *)&K256[4 * (I)]));    \
        st1 = _mm_sha256rnds2_epu32(st1, st0, msg);                                          \
        msg = _mm_shuffle_epi32(msg, 0x0E);                                                  \
        st0 = _mm_sha256rnds2_epu32(st0, st1, msg);                                          \
    }
// X_i = msg2(msg1(X_{i-4}, X_{i-3}) + alignr(X_{i-1}, X_{i-2}, 4), X_{i-1})
#define SHA_SCHED(Xi4, Xi3, Xi2, Xi1) \
    Xi4 = _mm_sha256msg2_epu32(_mm_add_epi32(_mm_sha256msg1_epu32(Xi4, Xi3), _mm_alignr_epi8(Xi1, Xi2, 4)), Xi1)
        w0 = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i *)(data + 0)), MASK);
        SHA_ROUNDS(w0, 0);
        w1 = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i *)(data + 16)), MASK);
        SHA_ROUNDS(w1, 1);
        w2 = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i *)(data + 32)), MASK);
        SHA_ROUNDS(w2, 2);
        w3 = _mm_shuffle_epi8(_mm_loadu_si128((const __m128i *)(data + 48)), MASK);
        SHA_ROUNDS(w3, 3);
        for (int i = 4; i < 16; i += 4) {
            SHA_SCHED(w0, w1, w2, w3); SHA_ROUNDS(w0, i);
            SHA_SCHED(w1, w2, w3, w0); SHA_ROUNDS(w1, i + 1);
            SHA_SCHED(w2, w3, w0, w1); SHA_ROUNDS(w2, i + 2);
            SHA_SCHED(w3, w0, w1, w2); SHA_ROUNDS(w3, i + 3);
        }
#undef SHA_ROUNDS
#undef SHA_SCHED
        st0 = _mm_add_epi32(st0, abef);
        st1 = _mm_add_epi32(st1, cdgh);
    }
    tmp = _mm_shuffle_epi32(st0, 0x1B);            // FEBA
    st1 = _mm_shuffle_epi32(st1, 0xB1);            // DCHG
    st0 = _mm_blend_epi16(tmp, st1, 0xF0);         // DCBA
    st1 = _mm_alignr_epi8(st1, tmp, 8);            // HGFE
    _mm_storeu_si128((__m128i *)&s[0], st0);
    _mm_storeu_si128((__m128i *)&s[4], st1);
}

bool cpu_has_sha() {
    unsigned a = 0, b = 0, c = 0, d = 0;
    if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
    const bool sha = (b >> 29) & 1u;
    __get_cpuid(1, &a, &b, &c, &d);
    const bool sse41 = (c >> 19) & 1u, ssse3 = (c >> 9) & 1u;
    return sha && sse41 && ssse3;
}

int g_force_portable = 0;

struct Sha256 {
    uint32_t s[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a, 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    uint8_t buf[64];
    size_t nbuf = 0;
    uint64_t total = 0;
    void (*blocks)(uint32_t *, const uint8_t *, size_t);
    Sha256() { blocks = (!g_force_portable && cpu_has_sha()) ? sha256_blocks_shani : sha256_blocks_portable; }
    void update(const void *p, size_t n) {
        const uint8_t *d = static_cast<const uint8_t *>(p);
        total += n;
        if (nbuf) {
            const size_t take = n < 64 - nbuf ? n : 64 - nbuf;
            std::memcpy(buf + nbuf, d, take);
            nbuf += take;
            d += take;
            n -= take;
            if (nbuf == 64) {
                blocks(s, buf, 1);
                nbuf = 0;
            }
        }
        if (n >= 64) {
            blocks(s, d, n / 64);
            d += n & ~size_t(63);
            n &= 63;
        }
        if (n) {
            std::memcpy(buf, d, n);
            nbuf = n;
        }
    }
    void hex(char out[65]) {
        const uint64_t bits = total * 8;
        const uint8_t pad = 0x80;
        update(&pad, 1);
        const uint8_t zero[64] = {0};
        update(zero, (nbuf <= 56) ? 56 - nbuf : 120 - nbuf);
        uint8_t len[8];
        for (int i = 0; i < 8; ++i) len[i] = (uint8_t)(bits >> (56 - 8 * i));
        update(len, 8);
        static const char *hx = "0123456789abcdef";
        for (int i = 0; i < 8; ++i)
            for (int b = 0; b < 4; ++b) {
                const uint8_t v = (uint8_t)(s[i] >> (24 - 8 * b));
                out[8 * i + 2 * b] = hx[v >> 4];
                out[8 * i + 2 * b + 1] = hx[v & 15];
            }
        out[64] = 0;
    }
};

// ------------------------------------------------------ chunked formatting

struct Chunk {
    int64_t l0, l1;                  // loops [l0, l1)
    char *data = nullptr;            // points into the persistent chunk pool
    size_t size = 0;
    std::atomic<bool> ready{false};
};

// Persistent per-chunk output buffers: reused across calls so the formatting
// threads do not page-fault fresh allocations every time (one digest at a time).
std::mutex g_pool_mu;
std::vector<std::unique_ptr<char[]>> g_pool;
std::vector<size_t> g_pool_cap;

char *pool_buffer(size_t k, size_t bound) {
    if (g_pool_cap[k] < bound) {
        g_pool[k].reset(new char[bound + bound / 4]);
        g_pool_cap[k] = bound + bound / 4;
    }
    return g_pool[k].get();
}

void pool_reserve(size_t n) {
    if (g_pool.size() < n) {
        g_pool.resize(n);
        g_pool_cap.resize(n, 0);
    }
}

bool all_finite(const double *a, int64_t n) {
    for (int64_t k = 0; k < n; ++k)
        if (!std::isfinite(a[k])) return false;
    return true;
}

struct Job {
    const double *coeffs, *t;
    const int64_t *off;
    const uint8_t *closed;
    const double *const *vptr = nullptr;  // per-loop vertex rows of closed polylines (coeffs/t unused)
    // streamed input (lc_model_digest_polylines_stream): loops [0, *ready) of vptr / off
    // are filled; a negative value aborts the digest
    const volatile int64_t *ready = nullptr;
    std::atomic<bool> aborted{false}, null_loop{false};
    std::vector<Chunk> chunks;
    std::atomic<int64_t> next{0};
    bool check_finite = false;           // digest: validate the chunk's coefficients in the worker
    std::atomic<bool> nonfinite{false};
    std::mutex mu;
    std::condition_variable cv;

    void format(Chunk &c) {
        if (vptr) {
            format_vertices(c);
            return;
        }
        size_t bound = 1;
        std::vector<uint8_t> poly((size_t)(c.l1 - c.l0));
        for (int64_t l = c.l0; l < c.l1; ++l) {
            const int64_t m = off[l + 1] - off[l];
            poly[l - c.l0] = loop_is_polyline(coeffs + 12 * off[l], t + 2 * off[l], m);
            bound += loop_bound(m, poly[l - c.l0]) + 1;
        }
        if (check_finite && !all_finite(coeffs + 12 * off[c.l0], 12 * (off[c.l1] - off[c.l0])))
            nonfinite.store(true);
        c.data = pool_buffer((size_t)(&c - chunks.data()), bound);
        char *p = c.data;
        for (int64_t l = c.l0; l < c.l1; ++l) {
            if (l) *p++ = ',';
            p = put_loop(p, coeffs + 12 * off[l], t + 2 * off[l], off[l + 1] - off[l], closed ? closed[l] != 0 : true,
                         poly[l - c.l0]);
        }
        c.size = (size_t)(p - c.data);
        {
            std::lock_guard<std::mutex> g(mu);
            c.ready.store(true, std::memory_order_release);
        }
        cv.notify_all();
    }

    // streamed input: wait until the chunk's loops are filled (or the caller aborts)
    bool wait_input(const Chunk &c) {
        if (!ready) return true;
        for (int spins = 0;; ++spins) {   // the caller publishes a piece every ~0.1 ms: poll, then sleep
            const int64_t r = *ready;
            if (r < 0) return false;
            if (r >= c.l1) break;
            if (spins > 16) std::this_thread::sleep_for(std::chrono::microseconds(20));
        }
        std::atomic_thread_fence(std::memory_order_acquire);
        for (int64_t l = c.l0; l < c.l1; ++l)
            if (off[l + 1] > off[l] && !vptr[l]) return null_loop.store(true), false;
        return true;
    }

    void format_vertices(Chunk &c) {
        if (!wait_input(c)) {   // nothing to format: the hasher stops at this chunk
            aborted.store(true);
            c.size = 0;
            {
                std::lock_guard<std::mutex> g(mu);
                c.ready.store(true, std::memory_order_release);
            }
            cv.notify_all();
            return;
        }
        size_t bound = 1;
        for (int64_t l = c.l0; l < c.l1; ++l) bound += loop_bound(off[l + 1] - off[l], true) + 1;
        bool fin = true;
        if (check_finite)
            for (int64_t l = c.l0; l < c.l1 && fin; ++l) fin = all_finite(vptr[l], 3 * (off[l + 1] - off[l]));
        if (!fin) nonfinite.store(true);
        c.data = pool_buffer((size_t)(&c - chunks.data()), bound);
        char *p = c.data;
        for (int64_t l = c.l0; l < c.l1; ++l) {
            if (l) *p++ = ',';
            p = put_loop_vertices(p, vptr[l], off[l + 1] - off[l]);
        }
        c.size = (size_t)(p - c.data);
        {
            std::lock_guard<std::mutex> g(mu);
            c.ready.store(true, std::memory_order_release);
        }
        cv.notify_all();
    }

    void worker() {
        for (;;) {
            const int64_t k = next.fetch_add(1);
            if (k >= (int64_t)chunks.size()) return;
            format(chunks[k]);
        }
    }

    void wait(Chunk &c) {
        if (c.ready.load(std::memory_order_acquire)) return;
        std::unique_lock<std::mutex> g(mu);
        cv.wait(g, [&] { return c.ready.load(std::memory_order_acquire); });
    }
};

// Split loops into chunks of ~target segments each.
void make_chunks(Job &job, int64_t L, int64_t M, int64_t target) {
    int64_t l = 0;
    std::vector<std::pair<int64_t, int64_t>> r;
    while (l < L) {
        // the first chunks are small so the in-order hasher starts almost at once
        const int64_t want = r.size() < 4 ? target / 8 : target;
        int64_t e = l + 1;
        while (e < L && job.off[e] - job.off[l] < want) ++e;
        r.emplace_back(l, e);
        l = e;
    }
    job.chunks = std::vector<Chunk>(r.size());
    for (size_t k = 0; k < r.size(); ++k) {
        job.chunks[k].l0 = r[k].first;
        job.chunks[k].l1 = r[k].second;
    }
    (void)M;
}

// Streamed input: chunk boundaries by loop count (the offsets are not known yet).
void make_chunks_by_loops(Job &job, int64_t L, int64_t per_chunk) {
    std::vector<std::pair<int64_t, int64_t>> r;
    for (int64_t l = 0; l < L;) {
        const int64_t want = r.size() < 4 ? (per_chunk / 8 > 0 ? per_chunk / 8 : 1) : per_chunk;
        const int64_t e = l + want < L ? l + want : L;
        r.emplace_back(l, e);
        l = e;
    }
    job.chunks = std::vector<Chunk>(r.size());
    for (size_t k = 0; k < r.size(); ++k) {
        job.chunks[k].l0 = r[k].first;
        job.chunks[k].l1 = r[k].second;
    }
}

int resolve_threads(int nthreads) {
    if (nthreads <= 0) nthreads = (int)std::thread::hardware_concurrency();
    if (nthreads < 1) nthreads = 1;
    return nthreads > 64 ? 64 : nthreads;
}

}  // namespace

extern "C" {

LC_API int64_t lc_model_json_bound(const int64_t *loop_off, int64_t L) {
    size_t b = 16;
    for (int64_t l = 0; l < L; ++l) b += loop_bound(loop_off[l + 1] - loop_off[l], false) + 1;
    return (int64_t)b;
}

LC_API int64_t lc_model_json(const double *coeffs, const double *t, const int64_t *loop_off,
                             const uint8_t *closed, int64_t L, int nthreads, char *out, int64_t cap) {
    const int64_t M = L > 0 ? loop_off[L] : 0;
    if (!all_finite(coeffs, 12 * M)) return -1;
    Job job{coeffs, t, loop_off, closed};
    std::lock_guard<std::mutex> pool_lock(g_pool_mu);
    make_chunks(job, L, M, 16384);
    pool_reserve(job.chunks.size());
    std::vector<std::thread> th;
    for (int k = 0; k < resolve_threads(nthreads) - 1; ++k) th.emplace_back([&] { job.worker(); });
    job.worker();
    for (auto &x : th) x.join();
    static const char head[] = "{\"loops\":[", tail[] = "]}";
    int64_t need = (int64_t)sizeof head - 1 + (int64_t)sizeof tail - 1;
    for (auto &c : job.chunks) need += (int64_t)c.size;
    if (need > cap) return -2;
    int64_t n = 0;
    std::memcpy(out, head, sizeof head - 1);
    n += sizeof head - 1;
    for (auto &c : job.chunks) {
        std::memcpy(out + n, c.data, c.size);
        n += (int64_t)c.size;
    }
    std::memcpy(out + n, tail, sizeof tail - 1);
    return n + (int64_t)sizeof tail - 1;
}

static int digest_job(Job &job, int64_t L, int nthreads, char *hex_out) {
    static const bool stats = std::getenv("LC_DIGEST_STATS") != nullptr;
    using clk = std::chrono::steady_clock;
    const auto ms = [](clk::time_point a, clk::time_point b) {
        return std::chrono::duration<double, std::milli>(b - a).count();
    };
    const auto t_begin = clk::now();
    const int64_t M = L > 0 && !job.ready ? job.off[L] : 0;   // streamed: off is being filled
    job.check_finite = true;
    std::lock_guard<std::mutex> pool_lock(g_pool_mu);
    if (job.ready)
        make_chunks_by_loops(job, L, 64);   // ~4096 segments for chainmail-sized loops
    else
        make_chunks(job, L, M, 4096);
    pool_reserve(job.chunks.size());
    const int nt = resolve_threads(nthreads);
    std::vector<std::thread> th;
    // the calling thread hashes; by default two cores stay free of formatting
    // workers — the hasher's and the one driving the GPU pipeline beside it
    // (formatting needs a fraction of the hash time on the remaining cores)
    const int workers = nthreads > 0 ? (nt > 1 ? nt - 1 : 1) : (nt > 3 ? nt - 2 : 1);
    for (int k = 0; k < workers; ++k) th.emplace_back([&] { job.worker(); });
    const auto t_spawned = clk::now();
    Sha256 h;
    h.update("{\"loops\":[", 10);
    double t_wait = 0.0, t_hash = 0.0;
    for (auto &c : job.chunks) {
        if (stats) {
            const auto t0 = clk::now();
            job.wait(c);
            const auto t1 = clk::now();
            h.update(c.data, c.size);
            t_wait += ms(t0, t1);
            t_hash += ms(t1, clk::now());
        } else {
            job.wait(c);
            h.update(c.data, c.size);
        }
        if (job.aborted.load()) break;
    }
    h.update("]}", 2);
    const auto t_hashed = clk::now();
    for (auto &x : th) x.join();
    const auto t_joined = clk::now();
    if (stats)
        std::fprintf(stderr,
                     "lc_model_digest: threads %d chunks %zu setup %.2f wait %.2f hash %.2f join %.2f total %.2f ms\n",
                     nt, job.chunks.size(), ms(t_begin, t_spawned), t_wait, t_hash, ms(t_hashed, t_joined),
                     ms(t_begin, t_joined));
    if (job.null_loop.load()) return -2;
    if (job.aborted.load()) return -3;
    if (job.nonfinite.load()) return -1;
    h.hex(hex_out);
    return 0;
}

LC_API int lc_model_digest(const double *coeffs, const double *t, const int64_t *loop_off, const uint8_t *closed,
                           int64_t L, int nthreads, char *hex_out) {
    Job job{coeffs, t, loop_off, closed};
    return digest_job(job, L, nthreads, hex_out);
}

LC_API int lc_model_digest_polylines(const double *const *loop_verts, const int64_t *loop_off, int64_t L,
                                     int nthreads, char *hex_out) {
    for (int64_t l = 0; l < L; ++l)
        if (loop_off[l + 1] > loop_off[l] && !loop_verts[l]) return -2;
    Job job{nullptr, nullptr, loop_off, nullptr};
    job.vptr = loop_verts;
    return digest_job(job, L, nthreads, hex_out);
}

LC_API int lc_model_digest_polylines_stream(const double *const *loop_verts, const int64_t *loop_off, int64_t L,
                                            const int64_t *ready, int nthreads, char *hex_out) {
    if (!ready || (L > 0 && (!loop_verts || !loop_off))) return -2;
    Job job{nullptr, nullptr, loop_off, nullptr};
    job.vptr = loop_verts;
    job.ready = ready;
    return digest_job(job, L, nthreads, hex_out);
}

LC_API int lc_sha256_hex(const void *data, int64_t n, int force_portable, char *hex_out) {
    g_force_portable = force_portable;
    Sha256 h;
    h.update(data, (size_t)n);
    h.hex(hex_out);
    g_force_portable = 0;
    return cpu_has_sha() ? 1 : 0;
}

LC_API int lc_float_repr(double x, char *out) {
    char *e = put_repr(out, x);
    *e = 0;
    return (int)(e - out);
}

LC_API int64_t lc_float_repr_many(const double *x, int64_t n, int use_tochars, char *out, int64_t cap) {
    if (cap < 26 * n) return -1;
    char *p = out;
    for (int64_t k = 0; k < n; ++k) {
        p = use_tochars ? put_repr_tochars(p, x[k]) : put_repr(p, x[k]);
        *p++ = '\n';
    }
    return (int64_t)(p - out);
}

}  // extern "C"
