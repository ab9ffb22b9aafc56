// Host build of the product's neighbour enumerator (paper_2502_01659_b200/csrc/masks.cuh)
// so tests can compare it with the oracle on the CPU.  Prints, for each row, the sorted
// union of its pieces (repeats kept) and whether the pieces were disjoint.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "masks.cuh"

int main(int argc, char **argv)
{
    if (argc < 6) { fprintf(stderr, "usage: kind L a b c\n"); return 2; }
    ga::DevMask M{};
    M.kind = atoi(argv[1]);
    M.L = atoll(argv[2]);
    long long a = atoll(argv[3]), b = atoll(argv[4]);
    M.parts = atoi(argv[5]); // LongNet: 1 = multiset mixture, 2 = per-head offsets
    const int head = argc > 6 ? atoi(argv[6]) : 0;
    if (M.kind == ga::K_WINDOW) { M.w = a; M.r = b; M.m = (a - 1) / b; }
    if (M.kind == ga::K_BLOCK_DILATED) { M.seg = a; M.r = b; }
    if (M.kind == ga::K_LONGNET) {
        M.w0 = a; M.alpha = b; M.K = 0;
        if (a <= M.L) { long long s = a; while (s * b <= M.L) { s *= b; ++M.K; } }
    }
    for (int64_t i = 0; i < M.L; ++i) {
        std::vector<int64_t> v;
        int np = ga::num_pieces_h(M, i, head);
        for (int pc = 0; pc < np; ++pc) {
            ga::Piece P = ga::get_piece_h(M, i, pc, head);
            for (int64_t k = 0; k < P.count; ++k) v.push_back(ga::piece_at(P, k));
        }
        size_t n = v.size();
        std::sort(v.begin(), v.end());
        std::vector<int64_t> u = v;
        bool disjoint = std::unique(u.begin(), u.end()) == u.end();
        if (head == 0 && ga::degree(M, i) != (int64_t)n) disjoint = false;
        printf("%lld %d", (long long)i, disjoint ? 1 : 0);
        for (auto j : v) printf(" %lld", (long long)j);
        printf("\n");
    }
    return 0;
}
