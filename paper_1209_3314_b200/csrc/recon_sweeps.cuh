// recon_sweeps.cuh -- scan sweeps / seed scan / contract check (recon_sweeps.cu).
#pragma once
#include "iwpp_common.cuh"

namespace iwpp {
namespace recon {

// dirs: bit 0 = forward (west neighbour, K.115-126), bit 1 = backward (K.129-139)
// (changed: optional device flag set to 1 when a cell changed)
int sweep_rows(void *J, const void *I, int W, int H, int dtype, cudaStream_t st, int dirs = 3,
               unsigned long long *changed = nullptr);
// The reference's sequential passes, exactly (recon_passes.cu): mode 0 raster
// (K.38-74), 1 anti-raster (K.77-112; seeds in anti-raster order when
// non-null), 2 / 3 column sweep forward / backward (K.142-190).  ctr[0] =
// changed, ctr[1] = seeds written.
int line_pass(void *J, const void *I, int W, int H, int dtype, int conn, int mode, int64_t *seeds,
              unsigned long long *ctr, cudaStream_t st);
// scratch: col_scratch_bytes(W, H) bytes of device memory
int sweep_cols(void *J, const void *I, int W, int H, int dtype, void *scratch, cudaStream_t st);
size_t col_scratch_bytes(int64_t W, int64_t H);
int seed_scan(const void *J, const void *I, int W, int H, int dtype, int conn, int64_t *out,
              unsigned long long *n_out, cudaStream_t st);
int check_le(const void *J, const void *I, size_t n, int dtype, unsigned long long *viol,
             cudaStream_t st);
// f32 <-> order-preserving int32 (in place allowed)
int f32_to_ord(const void *src, void *dst, size_t n, cudaStream_t st);
int ord_to_f32(const void *src, void *dst, size_t n, cudaStream_t st);

}  // namespace recon
}  // namespace iwpp
