// Device construction of the sliced-ELL views of a CSR pattern:
// the 3x3-block SELL-32 of vector problems (C3/C4) and the scalar SELL-32 of
// short-row stencils (C1/C2/C5). The host builders in linalg.py
// (_bsr3_from_host / _sell1_from_host) are the specification; these kernels
// produce bitwise the same arrays (tests/test_gpu_kernels.py compares them)
// in milliseconds instead of seconds of numpy per new pattern (C3: 3.5 s).
//
// Two passes, so the caller can size the slot arrays in between:
//   plan: per (block) row length and structure check -> per slice width ->
//         slice offsets sptr (exclusive scan, one block) and the slot count
//   fill: padding defaults for every slot, then the scatter of the real
//         (block) entries into slot order
#include <algorithm>

#include "common.cuh"

namespace rk {

constexpr int kSlice = 32;

// 3x3 structure of block row b: rows 3b..3b+2 have the same length, a
// multiple of 3, and their t-th column triple is (3c, 3c+1, 3c+2) with the
// same c in all three rows. Writes the block count of the row; raises *bad.
__global__ void k_bsr3_rows(int64_t nbr, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            int32_t* __restrict__ nb_per, int32_t* __restrict__ bad) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbr; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r0 = rp[3 * b], r1 = rp[3 * b + 1], r2 = rp[3 * b + 2], r3 = rp[3 * b + 3];
    const int64_t len = r1 - r0;
    bool ok = len % 3 == 0 && r2 - r1 == len && r3 - r2 == len;
    const int64_t nb = ok ? len / 3 : 0;
    for (int64_t t = 0; ok && t < nb; ++t) {
      const int32_t c0 = col[r0 + 3 * t];
      ok = c0 % 3 == 0 && col[r0 + 3 * t + 1] == c0 + 1 && col[r0 + 3 * t + 2] == c0 + 2;
      for (int a = 1; ok && a < 3; ++a) {
        const int64_t q = (a == 1 ? r1 : r2) + 3 * t;
        ok = col[q] == c0 && col[q + 1] == c0 + 1 && col[q + 2] == c0 + 2;
      }
    }
    nb_per[b] = (int32_t)nb;
    if (!ok) atomicOr(bad, 1);
  }
}

// Scalar rows: length of every row; raises *bad when one exceeds max_len.
__global__ void k_sell_rows(int64_t n, const int32_t* __restrict__ rp, int32_t max_len, int32_t* __restrict__ lens,
                            int32_t* __restrict__ bad) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t len = rp[r + 1] - rp[r];
    lens[r] = len;
    if (len > max_len) atomicOr(bad, 1);
  }
}

// Slice offsets: sptr[s + 1] - sptr[s] = 32 * max(len of the slice's rows);
// one 1024-thread block, fixed-order scan; *nslot = sptr[nsl].
__global__ void __launch_bounds__(1024) k_slice_scan(int64_t rows, const int32_t* __restrict__ len,
                                                     int32_t* __restrict__ sptr, int64_t* __restrict__ nslot) {
  __shared__ int64_t part[1024];
  const int64_t nsl = (rows + kSlice - 1) / kSlice;
  const int64_t per = (nsl + blockDim.x - 1) / blockDim.x;
  const int64_t s0 = threadIdx.x * per, s1 = min(nsl, s0 + per);
  int64_t acc = 0;
  for (int64_t s = s0; s < s1; ++s) {
    int32_t w = 0;
    for (int64_t r = s * kSlice; r < min(rows, (s + 1) * kSlice); ++r) w = max(w, len[r]);
    acc += (int64_t)w * kSlice;
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // inclusive Hillis-Steele scan
    const int64_t v = threadIdx.x >= (unsigned)off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int64_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t s = s0; s < s1; ++s) {
    sptr[s] = (int32_t)run;
    int32_t w = 0;
    for (int64_t r = s * kSlice; r < min(rows, (s + 1) * kSlice); ++r) w = max(w, len[r]);
    run += (int64_t)w * kSlice;
  }
  if (threadIdx.x == blockDim.x - 1) {
    sptr[nsl] = (int32_t)part[blockDim.x - 1];
    *nslot = part[blockDim.x - 1];
  }
}

// Padding defaults: every slot points at a valid (block) column -- the lane's
// own (block) row, clamped -- and gathers nothing (perm = -1).
__global__ void k_slot_defaults(int64_t rows, int64_t nsl, const int32_t* __restrict__ sptr, int64_t nslot, int vals,
                                int32_t* __restrict__ scol, int32_t* __restrict__ perm) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nslot; q += (int64_t)gridDim.x * blockDim.x) {
    // slice of slot q: the last s with sptr[s] <= q (binary search)
    int64_t lo = 0, hi = nsl - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (sptr[mid] <= q) lo = mid;
      else hi = mid - 1;
    }
    const int64_t pos = q - sptr[lo];
    scol[q] = (int32_t)min(lo * kSlice + pos % kSlice, rows - 1);
    for (int e = 0; e < vals; ++e) perm[q * vals + e] = -1;
  }
}

// Real 3x3 blocks: slot = sptr[b / 32] + 32 t + b % 32 holds block t of block
// row b; its 9 values live in the slot row's 9 x 32 tile at
// 9 (slot - slot % 32) + 32 (3a + c) + slot % 32.
__global__ void k_bsr3_fill(int64_t nbr, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ nb_per, const int32_t* __restrict__ sptr,
                            int32_t* __restrict__ scol, int32_t* __restrict__ perm) {
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbr; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t first[3] = {rp[3 * b], rp[3 * b + 1], rp[3 * b + 2]};
    const int64_t base = sptr[b / kSlice] + b % kSlice;
    for (int64_t t = 0; t < nb_per[b]; ++t) {
      const int64_t slot = base + t * kSlice;
      scol[slot] = col[first[0] + 3 * t] / 3;
      const int64_t tile = 9 * (slot - slot % kSlice) + slot % kSlice;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) perm[tile + kSlice * (3 * a + c)] = (int32_t)(first[a] + 3 * t + c);
    }
  }
}

// Real scalar entries: slot = sptr[r / 32] + 32 t + r % 32 holds entry t of row r.
__global__ void k_sell_fill(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const int32_t* __restrict__ sptr, int32_t* __restrict__ scol, int32_t* __restrict__ perm) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t beg = rp[r], len = rp[r + 1] - beg;
    const int64_t base = sptr[r / kSlice] + r % kSlice;
    for (int64_t t = 0; t < len; ++t) {
      scol[base + t * kSlice] = col[beg + t];
      perm[base + t * kSlice] = (int32_t)(beg + t);
    }
  }
}

}  // namespace rk

namespace rkh {

int elementwise_grid(int64_t n);

int sell_plan(int64_t n, const int32_t* rp, const int32_t* col, int32_t bdim, int32_t max_len, int32_t* len_ws,
              int32_t* sptr, int64_t* nslot, int32_t* bad, cudaStream_t s) {
  RK_REQUIRE(n > 0 && rp && len_ws && sptr && nslot && bad, RK_ERR_ARG, "rk_sell_plan: bad arguments");
  RK_REQUIRE(bdim == 1 || bdim == 3, RK_ERR_ARG, "rk_sell_plan: bdim must be 1 or 3");
  RK_REQUIRE(bdim == 1 || (n % 3 == 0 && col), RK_ERR_DIMENSION, "rk_sell_plan: 3x3 blocks need n %% 3 == 0");
  const int64_t rows = n / bdim;
  cudaMemsetAsync(bad, 0, sizeof(int32_t), s);
  if (bdim == 3) {
    rk::k_bsr3_rows<<<elementwise_grid(rows), 256, 0, s>>>(rows, rp, col, len_ws, bad);
  } else {
    rk::k_sell_rows<<<elementwise_grid(rows), 256, 0, s>>>(rows, rp, max_len, len_ws, bad);
  }
  note_launch();
  rk::k_slice_scan<<<1, 1024, 0, s>>>(rows, len_ws, sptr, nslot);
  note_launch();
  return cuda_check("rk_sell_plan");
}

int sell_fill(int64_t n, const int32_t* rp, const int32_t* col, int32_t bdim, const int32_t* len_ws,
              const int32_t* sptr, int64_t nslot, int32_t* scol, int32_t* perm, cudaStream_t s) {
  RK_REQUIRE(n > 0 && rp && col && sptr && scol && perm && nslot >= 0, RK_ERR_ARG, "rk_sell_fill: bad arguments");
  RK_REQUIRE(bdim == 1 || bdim == 3, RK_ERR_ARG, "rk_sell_fill: bdim must be 1 or 3");
  const int64_t rows = n / bdim, nsl = (rows + rk::kSlice - 1) / rk::kSlice;
  if (nslot > 0) {
    rk::k_slot_defaults<<<elementwise_grid(nslot), 256, 0, s>>>(rows, nsl, sptr, nslot, bdim == 3 ? 9 : 1, scol,
                                                                perm);
    note_launch();
  }
  if (bdim == 3) {
    rk::k_bsr3_fill<<<elementwise_grid(rows), 256, 0, s>>>(rows, rp, col, len_ws, sptr, scol, perm);
  } else {
    rk::k_sell_fill<<<elementwise_grid(rows), 256, 0, s>>>(rows, rp, col, sptr, scol, perm);
  }
  note_launch();
  return cuda_check("rk_sell_fill");
}

}  // namespace rkh
