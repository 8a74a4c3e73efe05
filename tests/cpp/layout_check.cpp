// Host check of the packed split-product K layouts in kernels.h (tc_layout with
// 64-coordinate slices, tc6_layout): for every d, tc_pos / tc_elem are inverse
// bijections between the stored terms (hi / lo of aligned coordinates, the
// three products of remainder coordinates) and the non-padding K positions,
// every position < 16 ns, and tc_chunk_run agrees with tc_elem on every chunk
// it claims.  Built and run by
// tests/test_cpu_boundary.py (g++ against the CUDA headers, no GPU).
#include <cstdio>
#include <vector>

#include "kernels.h"

using namespace rrs;

int main() {
    int bad = 0;
    for (int d = 1; d <= 256; ++d) {
        const TcLayout L = tc_layout(d);
        std::vector<int> seen(16 * L.ns, 0);
        int entries = 0, aligned = 0;
        for (int c = 0; c < d; ++c) {
            const int ne = tc_entries(L, c);
            entries += ne;
            aligned += ne == 2;
            for (int e = 0; e < ne; ++e) {
                const int kk = tc_pos(L, e, c);
                int e2, c2;
                if (kk < 0 || kk >= 16 * L.ns) { ++bad; continue; }
                tc_elem(L, kk, e2, c2);
                if (e2 != e || c2 != c || seen[kk]++) ++bad;
            }
        }
        int used = 0;
        for (int kk = 0; kk < 16 * L.ns; ++kk) {
            int e, c;
            tc_elem(L, kk, e, c);
            used += c >= 0;
        }
        if (used != entries) ++bad;
        // the split products: every (coordinate, product) pair is formed by exactly one
        // MMA pairing of A and B K steps (kernels.h: (g, g), (g, Q+g), (Q+g, g), (2Q+i, 2Q+i))
        // -- aligned coordinates: hi/lo entries; remainder: entry p in both operands
        if (aligned % 16 != 0) ++bad;
        for (int cc = 0; cc < 2 * L.ns; ++cc) {
            bool lo;
            int c0;
            if (!tc_chunk_run(L, cc, lo, c0)) continue;
            for (int e = 0; e < 8; ++e) {
                int e2, c2;
                tc_elem(L, 8 * cc + e, e2, c2);
                if (e2 != (lo ? 1 : 0) || c2 != c0 + e || tc_entries(L, c2) != 2) ++bad;
            }
        }
        // symbolic MMA sweep: every (A, B) term pair the MMAs multiply, per coordinate
        // exactly {hi hi, hi lo, lo hi} and nothing else (zero padding on either side)
        std::vector<int> prod(3 * d, 0);
        for (int s = 0; s <= L.full; ++s) {
            const int q = s < L.full ? 4 : L.q16;
            const int nm = s < L.full ? TC_SLICE_MMA : 3 * L.q16 + L.rsteps;
            for (int i = 0; i < nm; ++i) {
                int sa, sb;
                tc_mma_steps(q, i, sa, sb);
                for (int k = 0; k < 16; ++k) {
                    const int ka = 16 * (TC_SLICE_NS * s + sa) + k, kb = 16 * (TC_SLICE_NS * s + sb) + k;
                    int ea, ca, eb, cb;
                    tc_elem(L, ka, ea, ca);
                    tc_elem(L, kb, eb, cb);
                    if (ca < 0 || cb < 0) continue;
                    if (ca != cb) { ++bad; continue; }
                    const bool al = tc_a_lo(L, ea, ca), bl = tc_b_lo(L, eb, cb);
                    if (al && bl) { ++bad; continue; }
                    ++prod[3 * ca + (al ? 2 : bl ? 1 : 0)];
                }
            }
        }
        for (int v : prod)
            if (v != 1) ++bad;
        for (int c = 0; c < d; ++c)
            if (tc_entries(L, c) == 3 && (tc_a_lo(L, 0, c) || tc_a_lo(L, 1, c) || !tc_a_lo(L, 2, c))) ++bad;
        if (d <= 64 && L.full != 0) ++bad;
        if (tc_block_bytes(d) != 4096 * L.ns) ++bad;
        if (L.ns != 8 * L.full + 2 * L.q16 + L.rsteps || L.nmma != 12 * L.full + 3 * L.q16 + L.rsteps) ++bad;
    }
    for (int d = 1; d <= 64; ++d) {
        const Tc6Layout L = tc6_layout(d);
        std::vector<int> seen(16 * L.ns, 0);
        for (int c = 0; c < d; ++c)
            for (int p = 0; p < 6; ++p) {
                const int kk = tc6_pos(L, p, c);
                int p2, c2;
                if (kk < 0 || kk >= 16 * L.ns) { ++bad; continue; }
                tc6_elem(L, kk, p2, c2);
                if (p2 != p || c2 != c || seen[kk]++) ++bad;
            }
    }
    const int at[6] = {0, 0, 1, 0, 2, 1}, bt[6] = {0, 1, 0, 2, 0, 1};
    for (int p = 0; p < 6; ++p)
        if (tc6_a_term(p) != at[p] || tc6_b_term(p) != bt[p]) ++bad;
    std::printf("%s %d\n", bad ? "FAIL" : "OK", bad);
    return bad ? 1 : 0;
}
