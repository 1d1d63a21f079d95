// Device-side dispatch plan written by plan_kernel from the routing flows
// and read by dispatch / relayout / GEMM / colsum kernels. All arrays are
// device int32 inside one allocation owned by the layer.
#pragma once

#include <cstdint>

namespace fm {

struct PlanDev {
  int32_t* chunk_lo;        // [N][G]  first rank of dst's chunk in (me, e) rank space
  int32_t* chunk_cnt;       // [N][G]  flows[e][me][dst]
  int32_t* send_off;        // [N][G]  first dispatch-buffer row of (dst, e) (dst-major)
  int32_t* send_rows;       // [G]     rows sent to each dst
  int32_t* recv_rows;       // [G]     rows received from each src
  int32_t* local_index;     // [N]     local segment of expert e on this GPU, -1 if none (host-filled)
  int32_t* seg_start;       // [Nl]    first X_perm row of local expert li
  int32_t* seg_real;        // [Nl]    rows that carry tokens
  int32_t* seg_rows;        // [Nl]    rows padded to 128
  int32_t* mtile_prefix;    // [Nl+1]  exclusive prefix of 128-row tiles
  int32_t* recv_chunk_off;  // [G*Nl+1] a2a receive-buffer offset of (src, li)
  int32_t* recv_chunk_dst;  // [G*Nl]  X_perm row of that chunk's first row
  int32_t* totals;          // [4]     padded rows, units sent, units received
};

}  // namespace fm
