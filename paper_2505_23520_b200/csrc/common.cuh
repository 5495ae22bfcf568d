// Shared geometry and helpers for the AnchorAttention kernels.
//
// Index arithmetic is a bit-for-bit restatement of R/src/detail/geometry.hpp
// (R/ = /root/reference/proj/); every kernel derives its tile lists from
// these functions so host and device agree exactly.
#pragma once

#include <cstdint>

#include "../../include/anchorattn_capi.h"

#define AA_HD __host__ __device__ __forceinline__

namespace aa {

struct Geo {
    int64_t n, b_q, b_kv, step;

    AA_HD static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
    AA_HD int64_t q_blocks() const { return cdiv(n, b_q); }
    AA_HD int64_t kv_blocks() const { return cdiv(n, b_kv); }
    AA_HD int64_t group_rows() const { return step * b_q; }
    // geometry.hpp:36-38
    AA_HD int64_t groups() const { return cdiv(q_blocks(), step); }
    // geometry.hpp:40-47
    AA_HD int64_t row_begin(int64_t g) const { return g * step * b_q; }
    AA_HD int64_t row_end(int64_t g) const {
        const int64_t e = row_begin(g + 1);
        return e < n ? e : n;
    }
    // geometry.hpp:55-59
    AA_HD int64_t window_start_block(int64_t g) const {
        const int64_t rb = row_begin(g);
        if (rb < b_kv * 2) return 1;
        return rb / b_kv - 1;
    }
    // geometry.hpp:61-64
    AA_HD int64_t window_start(int64_t g) const {
        const int64_t w = window_start_block(g) * b_kv;
        return w < n ? w : n;
    }
    // geometry.hpp:66-69
    AA_HD int64_t middle_end(int64_t g) const {
        const int64_t w = window_start(g);
        const int64_t ib = b_kv < n ? b_kv : n;
        return w > ib ? w : ib;
    }
    AA_HD int64_t middle_len(int64_t g) const {
        const int64_t e = middle_end(g);
        return e > b_kv ? e - b_kv : 0;
    }
    // Capacity-layout slot base of group g (sum of middle_len over h < g).
    // middle_len(g) = max(0, min(wsb(g)*b_kv, n) - b_kv): closed form would
    // need care at the clamp; groups are few (<= a few thousand), loop is fine
    // on the host.  Device code receives offsets through a precomputed table.
    __host__ int64_t stripe_offset(int64_t g) const {
        int64_t off = 0;
        for (int64_t h = 0; h < g; ++h) off += middle_len(h);
        return off;
    }
    // geometry.hpp:79-85
    AA_HD int64_t covered_count_for_row(int64_t row) const {
        const int64_t init = b_kv < row + 1 ? b_kv : row + 1;
        const int64_t ws = window_start(row / (step * b_q));
        const int64_t window = row + 1 > ws ? row + 1 - ws : 0;
        return init + window;
    }
};

}  // namespace aa
