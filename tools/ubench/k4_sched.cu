// Print the compile-time K4 warp schedule (items per warp, DMMA load per warp) for one instantiation.
// nvcc -std=c++17 --expt-relaxed-constexpr -I paper_1904_06971_b200/csrc -DSG_MAX_P=4 -o /tmp/k4s tools/ubench/k4_sched.cu
#include "sg_tile_mma.cuh"
#include <cstdio>
using namespace sg;
int main() {
    const int nd = 3, P = 3, form = 0;
    const bool rat = false;
    const TileChoice tc = mma_tile(nd, P, form, rat);
    const MmaGeom M = mma_geom(nd, P, form, rat, tc.T0, tc.T1);
    const Tables T = make_tables(nd, form, rat);
    const int NW = mma_warps(nd, P, form, rat);
    static MmaTab S = mma_tab(nd, P, form, rat);
    printf("tile %dx%d NW %d NB %d KS %d KS3 %d MT %d NTY %d NG1 %d NG2 %d NU1 %d NCH %d CH %d smem %ld B\n", tc.T0, tc.T1, NW,
           mma_spec_nb(nd, form), M.KS, M.KS3, M.MT, M.NTY, M.NG1, M.NG2, M.NU1, M.NCH, M.CH, M.total * 8);
    for (int w = 0; w < NW; ++w) {
        long l1 = 0, l2 = 0, l3 = 0;
        printf("warp %2d:", w);
        for (int q = S.v[S.o_off1 + w]; q < S.v[S.o_off1 + w + 1]; ++q) {
            const int k = S.v[S.o_it1 + q], gk = k / (M.T0 * M.NC1);
            const int c = T.g1n[gk] * M.KS * M.MT * (M.NTY / M.NC1);
            l1 += c;
            printf(" p1[%d]=%d", k, c);
        }
        for (int q = S.v[S.o_off2 + w]; q < S.v[S.o_off2 + w + 1]; ++q) {
            const int k = S.v[S.o_it2 + q];
            const int c = g2_blocks(T, k / (M.T1 * M.T0)) * M.KS * M.MT * M.MT;
            l2 += c;
            printf(" p2[%d]=%d", k, c);
        }
        for (int q = S.v[S.o_off3 + w]; q < S.v[S.o_off3 + w + 1]; ++q) {
            const int c = (T.NF + f_npairs(T)) * M.KS3 * M.CH * M.MT;
            l3 += c;
        }
        printf("  | A %ld  B(phase3 per row plane) %ld\n", l1 + l2, l3);
    }
    return 0;
}
