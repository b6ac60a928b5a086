// shard.cu — pack / unpack of register sub-blocks for the global-qubit exchange of sharded states
// (sharded.py drives the schedule and the NCCL transport).
//
// A remap of j global qubits against local bit positions l_1..l_j moves, to partner p, the rows of
// the shard whose local bits l_i equal p's global bits k_i: a 1/2^j sub-block with j fixed row
// bits.  Sub-block row h (0 .. 2^n/2^j - 1, in increasing order) is row deposit(h, l) | fixval.
// pack gathers a contiguous range of sub-block rows (one staging chunk) into a flat buffer;
// unpack scatters a received chunk back.  Every row carries its B batch-innermost amplitudes, so
// with runs of 2^min(l) rows both sides stream coalesced 16-B elements; HBM-bound (2 x bytes).
#include <algorithm>

#include "engine.h"

namespace qbg {
namespace {

struct FixArgs {
    uint8_t pos[8];    // fixed local bit positions, ascending
    int nfix;
    uint64_t fixval;   // their values placed at pos (a row mask)
};

template <typename V, bool PACK>
__global__ void __launch_bounds__(256) k_shard_copy(V* __restrict__ st, V* __restrict__ buf, FixArgs f, uint64_t h0,
                                                    uint64_t count, int64_t B) {
    const uint64_t n = count * static_cast<uint64_t>(B);
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t e = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += stride) {
        const uint64_t h = e / static_cast<uint64_t>(B), b = e - h * static_cast<uint64_t>(B);
        const uint64_t row = deposit_zeros(h0 + h, f.pos, f.nfix) | f.fixval;
        V* s = st + row * static_cast<uint64_t>(B) + b;
        if (PACK)
            buf[e] = *s;
        else
            *s = buf[e];
    }
}

}  // namespace

void launch_shard_copy(const DevState& s, bool pack, const int* fix_pos, int nfix, uint64_t fix_val, uint64_t h0,
                       uint64_t count, void* buf) {
    if (nfix < 0 || nfix > 8) raise(QBG_ERR_VALIDATION, "shard pack: 0..8 fixed bits");
    FixArgs f{};
    f.nfix = nfix;
    int order[8];
    for (int i = 0; i < nfix; ++i) order[i] = i;
    for (int i = 0; i < nfix; ++i)  // ascending positions (insertion sort; j <= 8)
        for (int j = i + 1; j < nfix; ++j)
            if (fix_pos[order[j]] < fix_pos[order[i]]) std::swap(order[i], order[j]);
    for (int i = 0; i < nfix; ++i) {
        const int p = fix_pos[order[i]];
        if (p < 0 || p >= s.n || (i > 0 && p == f.pos[i - 1])) raise(QBG_ERR_RANGE, "shard pack: bad fixed bit position");
        f.pos[i] = static_cast<uint8_t>(p);
        if ((fix_val >> order[i]) & 1) f.fixval |= uint64_t{1} << p;
    }
    const uint64_t sub_rows = s.rows() >> nfix;
    if (h0 > sub_rows || count > sub_rows - h0) raise(QBG_ERR_RANGE, "shard pack: row range outside the sub-block");
    if (count == 0) return;
    const uint64_t n = count * static_cast<uint64_t>(s.B);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(num_sms()) * 16));
    LaunchScope ls(pack ? "shard_pack" : "shard_unpack", 2.0 * n * s.elem());
    if (s.dtype == QBG_C128) {
        if (pack)
            k_shard_copy<double2, true><<<grid, 256, 0, stream()>>>(static_cast<double2*>(s.ptr), static_cast<double2*>(buf), f, h0, count, s.B);
        else
            k_shard_copy<double2, false><<<grid, 256, 0, stream()>>>(static_cast<double2*>(s.ptr), static_cast<double2*>(buf), f, h0, count, s.B);
    } else {
        if (pack)
            k_shard_copy<float2, true><<<grid, 256, 0, stream()>>>(static_cast<float2*>(s.ptr), static_cast<float2*>(buf), f, h0, count, s.B);
        else
            k_shard_copy<float2, false><<<grid, 256, 0, stream()>>>(static_cast<float2*>(s.ptr), static_cast<float2*>(buf), f, h0, count, s.B);
    }
    QBG_CUDA(cudaGetLastError());
}

}  // namespace qbg
