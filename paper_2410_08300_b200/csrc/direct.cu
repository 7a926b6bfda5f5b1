// direct.cu -- dispatch of the `direct` algorithm (§II.B(d): "kernels are
// applied directly to the input without transforming the data").  The
// kernel and its design notes are in direct_impl.cuh; the tile-shape variants are compiled
// in direct_q2.cu / direct_q4.cu / direct_q8.cu.
#include "internal.h"

namespace ai3 {

template <int QG, int NKG>
cudaError_t launch_direct_qg(const DirectArgs& a, cudaStream_t st);

namespace {
constexpr int NT = 256;
}  // namespace

cudaError_t launch_direct(const DirectArgs& a, cudaStream_t st) {
    // 64 channels per CTA when the group has them (halves the staging per FFMA), else 32;
    // then the tile shape with the least padded area (ties: the widest rows)
    const int nkg = a.Kg > 32 ? 8 : 4;
    const int pt = NT / nkg;
    int best = 8;
    long long best_area = -1;
    for (int qg : {8, 4, 2}) {
        const long long tq = 8 * qg, tp = pt / qg;
        const long long area = ((a.P + tp - 1) / tp) * tp * ((a.Q + tq - 1) / tq) * tq;
        if (best_area < 0 || area < best_area) { best = qg; best_area = area; }
    }
    if (nkg == 8) {
        if (best == 8) return launch_direct_qg<8, 8>(a, st);
        if (best == 4) return launch_direct_qg<4, 8>(a, st);
        return launch_direct_qg<2, 8>(a, st);
    }
    if (best == 8) return launch_direct_qg<8, 4>(a, st);
    if (best == 4) return launch_direct_qg<4, 4>(a, st);
    return launch_direct_qg<2, 4>(a, st);
}

}  // namespace ai3
