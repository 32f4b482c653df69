// ft_tables.cu -- host construction of the transition-class tables.
//
// Mirrors paper_2311_11740_b200/_tables.py (which is pinned to the reference
// classifier, contrib3d.py:76-135, by tests/test_tables.py); the ordering of
// classes is (stage rank, source type, destination type) in both.
#include <mutex>
#include <set>
#include <tuple>
#include <vector>

#include "ft_tables.h"

namespace ft {

static int popc(int x) { return __builtin_popcount(x); }

// Stage type of an active-slot mask, 3D (contrib3d.py:101-135).
static int type3(int mask)
{
    int n = popc(mask);
    if (n == 0) return -1;
    if (n == 1) return 0;
    if (n == 7) return 19;
    if (n == 8) return 20;
    int f = 0, e = 0, v = 0;
    int sel = n <= 4 ? mask : (~mask & 0xFF);
    for (int a = 0; a < 8; ++a)
        for (int b = a + 1; b < 8; ++b)
            if ((sel >> a & 1) && (sel >> b & 1)) {
                int d = popc(a ^ b);
                (d == 1 ? f : d == 2 ? e : v)++;
            }
    auto pair = [&](int base) { return f == 1 ? base : e == 1 ? base + 1 : v == 1 ? base + 2 : -2; };
    auto triple = [&](int base) {
        if (f == 2 && e == 1 && v == 0) return base;
        if (f == 1 && e == 1 && v == 1) return base + 1;
        if (f == 0 && e == 3 && v == 0) return base + 2;
        return -2;
    };
    switch (n) {
    case 2: return pair(1);
    case 3: return triple(4);
    case 4:
        if (f == 4 && e == 2 && v == 0) return 7;
        if (f == 3 && e == 3 && v == 0) return 8;
        if (f == 3 && e == 2 && v == 1) return 9;
        if (f == 2 && e == 3 && v == 1) return 10;
        if (f == 2 && e == 2 && v == 2) return 11;
        if (f == 0 && e == 6 && v == 0) return 12;
        return -2;
    case 5: return triple(13);
    case 6: return pair(16);
    }
    return -2;
}

// 2D stage type: q1 q2 qd q3 q4 (contrib2d.py:36); diagonal iff the two
// active slots sum to 3 (NW+SE, NE+SW; contrib2d.py:224).
static int type2(int mask)
{
    int n = popc(mask);
    if (n == 0) return -1;
    if (n == 1) return 0;
    if (n == 2) return (mask == 0x9 || mask == 0x6) ? 2 : 1;
    return n == 3 ? 3 : 4;
}

static void build(int ndim, Tables& t)
{
    const int S = ndim == 3 ? 8 : 4;
    auto typ = ndim == 3 ? type3 : type2;
    std::set<std::tuple<int, int, int>> pairs;
    for (int mask = 0; mask < (1 << S) - 1; ++mask)
        for (int s = 0; s < S; ++s)
            if (!(mask >> s & 1)) pairs.insert({popc(mask), typ(mask), typ(mask | 1 << s)});
    t.S = S;
    t.n_classes = (int)pairs.size();
    std::vector<std::tuple<int, int, int>> ord(pairs.begin(), pairs.end());
    for (int c = 0; c < t.n_classes; ++c) {
        t.src[c] = std::get<1>(ord[c]);
        t.dst[c] = std::get<2>(ord[c]);
    }
    for (int i = 0; i < (1 << S) * S; ++i) t.step[i] = -1;
    for (int mask = 0; mask < (1 << S) - 1; ++mask)
        for (int s = 0; s < S; ++s)
            if (!(mask >> s & 1)) {
                int a = typ(mask), b = typ(mask | 1 << s);
                for (int c = 0; c < t.n_classes; ++c)
                    if (t.src[c] == a && t.dst[c] == b) t.step[mask * S + s] = c;
            }
}

const Tables& tables(int ndim)
{
    static Tables t2, t3;
    static std::once_flag once;
    std::call_once(once, [] {
        build(2, t2);
        build(3, t3);
    });
    return ndim == 3 ? t3 : t2;
}

}  // namespace ft

extern "C" int ft_tables(int32_t ndim, int32_t* step, int32_t* src, int32_t* dst)
{
    if (ndim != 2 && ndim != 3) return FT_ERR_ARG;
    const ft::Tables& t = ft::tables(ndim);
    if (step)
        for (int i = 0; i < (1 << t.S) * t.S; ++i) step[i] = t.step[i];
    for (int c = 0; c < t.n_classes; ++c) {
        if (src) src[c] = t.src[c];
        if (dst) dst[c] = t.dst[c];
    }
    return FT_OK;
}

extern "C" int ft_class_weights(int32_t ndim, const int64_t* eighths, int64_t* out)
{
    if ((ndim != 2 && ndim != 3) || !eighths || !out) return FT_ERR_ARG;
    const ft::Tables& t = ft::tables(ndim);
    for (int c = 0; c < t.n_classes; ++c)
        out[c] = eighths[t.dst[c]] - (t.src[c] >= 0 ? eighths[t.src[c]] : 0);
    return FT_OK;
}

extern "C" const char* ft_version(void) { return "fieldtopo-b200 0.1.0 (sm_100a)"; }
