// k_layout.cu -- K0: device layout of this rank's resident lists (load time,
// not timed). P:339-341 (index splitter), P:423 ("clusters are stored
// contiguously to enable high-bandwidth access").
//
// Each resident list is cut into groups of 32 vectors (the last one padded).
// Group g holds, for lane v (= vector v of the group):
//   codes: [mpad*nbits/128 chunks][32 lanes][16 bytes] -- one coalesced
//          512-byte LDG.128 per chunk per warp; lane v's sub-codes are
//          ROTATED: slot s = 32r + t holds sub-code j = 32r + (v ^ t) (0 for
//          j >= m), the order the scan's conflict-free LUT gathers consume
//          them in. A slot is a byte (8-bit codes; 4-bit codes in pair
//          mode: slot j' = packed byte j' = sub-codes 2j', 2j'+1) or a nibble
//          (4-bit nibble mode: slot s is the low nibble of byte s/2 for even s).
//   bias:  b_v = ||yhat_v||^2 + 2 <c_l, yhat_v> computed in fp64, rounded to
//          fp32 (+inf for padding slots, so they never enter a top-k);
//          ||yhat_v||^2 without residual codes, 0 for the inner-product
//          metric (NEXT-3).
//   ids:   int64 id (-1 for padding).
#include <cfloat>

#include "vlr_device.cuh"
#include "vlr_internal.cuh"

namespace vlr {

// sub-code j of an input code row (nbits 8: byte j; 4: nibble j, low first)
__device__ __forceinline__ uint32_t in_code(const uint8_t* row, int j, int nbits) {
  return nbits == 8 ? row[j] : (row[j >> 1] >> (4 * (j & 1))) & 15u;
}

__global__ void k_layout(int d, int m, int mpad, int dsub, int nbits, int code_m, int code_bits, int metric,
                         int by_residual, int n_local,
                         long long n_slots,
                         const int64_t* __restrict__ gbase, const int64_t* __restrict__ vbase,
                         const int32_t* __restrict__ lglob, const uint8_t* __restrict__ scodes,
                         const int64_t* __restrict__ sids, const float* __restrict__ C, const float* __restrict__ Y,
                         uint8_t* __restrict__ codes, float* __restrict__ bias, int64_t* __restrict__ ids) {
  for (long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x; slot < n_slots;
       slot += (long long)gridDim.x * blockDim.x) {
    const long long grp = slot >> 5;
    const int lane = (int)(slot & 31);
    int lo = 0, hi = n_local;  // gbase[lo] <= grp < gbase[hi]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (gbase[mid] <= grp) lo = mid; else hi = mid;
    }
    const int list = lo;
    const long long pos = (grp - gbase[list]) * 32 + lane;
    const long long len = vbase[list + 1] - vbase[list];
    const int ksub = 1 << nbits;
    const int nchunk = mpad * code_bits / 128;  // 16-byte chunks per lane
    const long long rowb = ((long long)m * nbits + 7) / 8;
    uint4* gdst = reinterpret_cast<uint4*>(codes + grp * 32LL * (mpad * code_bits / 8));
    if (pos < len) {
      const long long v = vbase[list] + pos;
      const uint8_t* src = scodes + v * rowb;
      const float* c = C + (size_t)lglob[list] * d;
      double b = 0.0;
      if (metric == 0) {
        for (int j = 0; j < m; ++j) {
          const float* y = Y + ((size_t)j * ksub + in_code(src, j, nbits)) * dsub;
          for (int u = 0; u < dsub; ++u) {
            const double yy = (double)y[u];
            b += yy * yy + (by_residual ? 2.0 * (double)c[j * dsub + u] * yy : 0.0);
          }
        }
      }
      bias[slot] = (float)b;
      ids[slot] = sids[v];
      // slots: sub-codes (8-bit codes, 4-bit nibble mode) or packed bytes (4-bit pair mode, code_m = ceil(m/2))
      const int per_byte = 8 / code_bits;  // slots per byte
      for (int ch = 0; ch < nchunk; ++ch) {
        uint32_t w[4];
        for (int q = 0; q < 4; ++q) {
          uint32_t word = 0;
          for (int bb = 0; bb < 4; ++bb) {
            uint32_t byte = 0;
            for (int h = 0; h < per_byte; ++h) {
              const int s = (ch * 16 + q * 4 + bb) * per_byte + h;  // slot
              const int j = 32 * (s >> 5) + (lane ^ (s & 31));
              byte |= (j < code_m ? in_code(src, j, code_bits) : 0u) << (code_bits * h);
            }
            word |= byte << (8 * bb);
          }
          w[q] = word;
        }
        gdst[ch * 32 + lane] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    } else {
      bias[slot] = CUDART_INF_F;
      ids[slot] = -1;
      for (int ch = 0; ch < nchunk; ++ch) gdst[ch * 32 + lane] = make_uint4(0, 0, 0, 0);
    }
  }
}

cudaError_t launch_layout(const DeviceIndex& ix, const uint8_t* stage_codes, const int64_t* stage_ids,
                          const int64_t* vbase, const int32_t* lglob, cudaStream_t s) {
  const long long n_slots = ix.n_groups * 32;
  if (n_slots == 0) return cudaSuccess;
  const int threads = 256;
  long long blocks = (n_slots + threads - 1) / threads;
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_layout<<<(int)blocks, threads, 0, s>>>(ix.d, ix.m, ix.mpad, ix.dsub, ix.nbits, ix.code_m, ix.code_bits,
                                           ix.metric, ix.by_residual,
                                           ix.n_local, n_slots, ix.gbase, vbase, lglob, stage_codes, stage_ids,
                                           ix.centroids, ix.codebooks, ix.codes, ix.bias, ix.ids);
  return cudaGetLastError();
}

}  // namespace vlr
