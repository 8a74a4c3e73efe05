// Host check of the packed split-product K layouts in kernels.h (tc_layout with
// 64-coordinate slices, tc6_layout): for every d, tc_pos / tc_elem are inverse
// bijections onto the non-padding K positions, every position < 16 ns, and
// tc_chunk_run agrees with tc_elem on every chunk it claims.  Built and run by
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
        for (int c = 0; c < d; ++c)
            for (int p = 0; p < 3; ++p) {
                const int kk = tc_pos(L, p, c);
                int p2, c2;
                if (kk < 0 || kk >= 16 * L.ns) { ++bad; continue; }
                tc_elem(L, kk, p2, c2);
                if (p2 != p || c2 != c || seen[kk]++) ++bad;
            }
        int used = 0;
        for (int kk = 0; kk < 16 * L.ns; ++kk) {
            int p, c;
            tc_elem(L, kk, p, c);
            used += c >= 0;
        }
        if (used != 3 * d) ++bad;
        for (int cc = 0; cc < 2 * L.ns; ++cc) {
            int p, c0;
            if (!tc_chunk_run(L, cc, p, c0)) continue;
            for (int e = 0; e < 8; ++e) {
                int p2, c2;
                tc_elem(L, 8 * cc + e, p2, c2);
                if (p2 != p || c2 != c0 + e) ++bad;
            }
        }
        if (d <= 64 && L.full != 0) ++bad;
        if (tc_block_bytes(d) != 4096 * L.ns) ++bad;
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
