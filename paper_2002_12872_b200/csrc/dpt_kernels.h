// dpt_kernels.h -- internal launch API of the CUDA kernels (host side).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "dpt_device.cuh"

namespace dpt {

// dense_step.cu (K1)
int make_tmap_rowmajor(CUtensorMap* out, const double* base, int64_t dim0, int64_t dim1, int64_t ld,
                       int box1);
int dense_cfg_for(int64_t n, int64_t rows);
int dense_tile_n(int cfg);
int dense_tile_m(int cfg);
cudaError_t launch_delta_image(const double* src, int64_t n, int cx, int transposed, double* dst, int64_t ldd,
                               cudaStream_t st);
int dense_step_ntiles(int64_t rows, int ntn, int cfg);
int dense_init_ntiles(int64_t rows, int ntn, int cplx);
cudaError_t launch_dense_step(const DevSolve& s, const CUtensorMap* amaps, const CUtensorMap* dmap,
                              const double* delta, int cfg, cudaStream_t st);
cudaError_t launch_dense_init(const DevSolve& s, const double* delta, int cfg, cudaStream_t st);

// sparse_step.cu (K2: CSR full map; K3: CSR / dense row map)
struct DevCsr {
  const int64_t* rowptr;  // [n+1]
  const int32_t* cols;    // [nnz]
  const double* vals;     // [nnz]
  int64_t nnz;
};
// SELL-32 image of Delta for K2 (built by build_sell in solver.cu)
struct DevSell {
  const int32_t* cols;      // [padded]
  const double* vals;       // [padded]
  const int64_t* slice_off; // [nslices + 1], multiples of 32
  const int32_t* lane_col;  // [nslices * 32] row of Delta (output column j) per lane, -1 = padding
  const int32_t* lane_len;  // [nslices * 32]
  const int64_t* pos_of;    // [n] lane index of row j
  int64_t nslices;
  const int32_t* perm;      // [n] shared-memory position of column k (bank balance), null = identity
  const int32_t* inv;       // [npad] column at position p (-1 = unused), null = identity
  int64_t npad;             // staged row length in positions (>= n)
  // K2's shared-memory kernel reads a packed copy (launch_sell_pack), null when not built:
  const uint16_t* cols16;   // [padded] the columns as 16-bit positions, trip-major: entry (step q, lane L)
                            //          of a slice at slice_off + (q / 4) * 128 + 4 L + (q & 3); 0xffff = bubble
  const int32_t* lane_pos;  // [nslices * 32] position of each lane's own column j (perm[j], or j), -1 = padding
  const double* lane_theta; // [nslices * 32] theta[j] of each lane's column
};
int csr_step_ntiles(int64_t rows, int64_t n);
int csr_ntn(int64_t n);
cudaError_t launch_csr_step(const DevSolve& s, const DevSell& d, cudaStream_t st);
// launch 1 from A_0 = I without the product (sparse_step.cu); scratch >= (rows + 4) * 8 bytes; the fold reads 1 tile
cudaError_t launch_csr_init(const DevSolve& s, const DevCsr& c, const DevSell& d, void* scratch, cudaStream_t st);

// row map (single vector): z slots are [nslots][n]
int single_mode(int dense, int uniform16);
int single_ntn(int64_t n, int mode);
int single_ntiles(int64_t n, int mode);
cudaError_t launch_single_step(const DevSolve& s, const DevCsr& d, const double* dense, int64_t row, int mode,
                               cudaStream_t st);
// uniform-16 CSR row map, launch 1 from z_0 = e_row without the gathers (single_u16.cu)
cudaError_t launch_single_u16_init(const DevSolve& s, const DevCsr& d, int64_t row, cudaStream_t st);

// complex_steps.cu (complex K2 / K3)
int csr_cplx_ntiles(int64_t rows, int64_t n);
cudaError_t launch_csr_step_cplx(const DevSolve& s, const DevSell& d, cudaStream_t st);
int single_cplx_ntiles(int64_t n, int dense, int u16);
// u16c_cols / u16c_vals: trip-major copy of a uniform-16 complex CSR (launch_u16c_build), or null
cudaError_t launch_single_cplx(const DevSolve& s, const DevCsr& d, const double* B, const int32_t* u16c_cols,
                               const double* u16c_vals, int64_t row, cudaStream_t st);
cudaError_t launch_u16c_build(const int32_t* cols, const double* vals, int64_t n, int32_t* ct, double* vt,
                              cudaStream_t st);

// fold.cu (K4)
int fold_blocks(int64_t rows);
cudaError_t launch_fold(const DevSolve& s, int ntiles_this, cudaStream_t st);
cudaError_t launch_decide(const DevSolve& s, cudaStream_t st);
cudaError_t launch_cycle(const DevSolve& s, int64_t elems, cudaStream_t st);
cudaError_t launch_identity(const DevSolve& s, cudaStream_t st);
// homotopy.cu: element-wise steps of the device homotopy_solve (row-major, cx = 1 | 2)
int dense_sk_grid(int cplx);          // stream-K K1: resident CTAs (persistent grid)
size_t dense_sk_part_doubles();       // stream-K K1: doubles per partial tile
cudaError_t launch_hom_stage_matrix(const double* D, const double* d, double lr, double li, int cx, int64_t n,
                                    int64_t ld, double* M, cudaStream_t st);
cudaError_t launch_hom_partition(const double* R, int64_t ld, double* dlev, double* Dp, int cx, int64_t n,
                                 cudaStream_t st);
cudaError_t launch_hom_normalise(const double* W, int64_t ld, double* a, int cx, int64_t n, unsigned* singular,
                                 cudaStream_t st);
cudaError_t launch_hom_densify(const int64_t* rp, const int32_t* cl, const double* vl, int cx, int64_t n, int64_t ld,
                               double* D, cudaStream_t st);
cudaError_t launch_hom_identity(double* W, int cx, int64_t n, int64_t ld, cudaStream_t st);
cudaError_t launch_hom_nonfinite(const double* a, int64_t count, unsigned* bad, cudaStream_t st);
// linalg.cu: library-free dense linear algebra of the device homotopy (row-major
// FP64, leading dims in doubles, complex interleaved when cx = 2)
cudaError_t launch_gemm_nt(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double alpha, double beta, double* Cm, int64_t ldc, cudaStream_t st);
cudaError_t launch_gemm_bop(int cx, bool trans, const double* S, int64_t lds, int64_t N, int64_t K, double* out,
                            int64_t ldo, cudaStream_t st);
cudaError_t launch_lu_factor(int cx, double* A, int64_t lda, int64_t n, int64_t* piv, int* info, double* scratch,
                             int* launches, cudaStream_t st);
cudaError_t launch_lu_solve(int cx, const double* A, int64_t lda, int64_t n, double* X, int64_t ldx, int64_t nrhs,
                            double* scratch, int* launches, cudaStream_t st);
cudaError_t launch_gather_rows(const double* src, int64_t ld, const int64_t* perm, int64_t n, int64_t width,
                               double* dst, cudaStream_t st);
int64_t lu_max_n(int cx);

// scan.cu: batched scan_domain, one warp per lambda cell (complex arithmetic in
// the reference's operation order).  All arrays complex interleaved unless noted.
struct ScanArgs {
  int64_t cells, res_re;
  int n, single, row, max_iter, win;
  int ring_smem;   // set by launch_scan: window ring in shared memory
  int warp_elems;  // set by launch_scan: complex elements of shared memory per warp
  double tol, res_tol, div_thr;
  const double* d;        // [n] levels
  const double* delta;    // [n*n] Delta (row map: w = Delta z)
  const double* delta_t;  // [n*n] Delta^T (full map: P = A Delta^T)
  const double* theta;    // [n*n] 1 / (d_i - d_j) (host std::complex division)
  const double* gap_row;  // [n] 1 / (d_row - d_m)
  const double* re_at;    // [res_re] real grid coordinates
  const double* im_at;    // [res_im] imaginary grid coordinates
  const double* ramp;     // [max_iter + 1] 1 - alpha^(k-1) (host std::pow), or null
  double* ring;           // per-warp cycle window ring
  uint8_t* classes;       // [cells] CellClass
  int32_t* iterations;    // [cells]
};
int scan_max_n(int single);
int64_t scan_tiny_threads(const ScanArgs& a);  // > 0: n <= 3 runs one thread per cell (ring per thread)
cudaError_t launch_scan(const ScanArgs& a, int warps_total, cudaStream_t st);

// sell_build.cu: K2's SELL-32 image built on the device from the CSR in HBM
cudaError_t launch_sell_perm(const int64_t* rp, int64_t n, int32_t* lane_col, int32_t* lane_len, int64_t* pos_of,
                             cudaStream_t st);
cudaError_t launch_sell_widths(const int64_t* rp, const int32_t* cl, int64_t nslices, const int32_t* lane_col, int G,
                               int sched, const int32_t* perm, int64_t* widths, cudaStream_t st);
cudaError_t launch_sell_scan(int64_t* widths, int64_t nslices, int64_t* total, cudaStream_t st);
cudaError_t launch_sell_fill(const int64_t* rp, const int32_t* cl, const double* vl, int cx, int64_t nslices,
                             const int32_t* lane_col, int G, int sched, const int32_t* perm, const int64_t* off,
                             int32_t* s_cols, double* s_vals, cudaStream_t st);
// column relabelling for bank balance (real K2): pos / inv permutation, padded staged-row length
size_t relabel_smem_bytes(int64_t nslices);
cudaError_t launch_sell_pack(const int32_t* s_cols, const int64_t* off, int64_t nslices, const int32_t* lane_col,
                             const int32_t* perm, const double* theta, uint16_t* cols16, int32_t* lane_pos,
                             double* lane_theta, cudaStream_t st);
cudaError_t launch_csr_order_check(const int64_t* rp, const int32_t* cl, int64_t n, int32_t* flag, cudaStream_t st);
cudaError_t launch_relabel(const int64_t* rp, const int32_t* cl, int64_t n, int64_t nnz, int64_t nslices,
                           const int64_t* slot_of, int cap, int passes, int32_t* scratch, int32_t* bank, int32_t* pos,
                           int32_t* inv, int64_t npad_alloc, int32_t* npad_out, cudaStream_t st);
int csr_staged_cols_max(int64_t n);  // longest staged row (positions) keeping K2's natural R; 0 = global gathers
// levels.cu: device-side setup scans (dominant selection, gap-row degeneracy, uniform CSR)
cudaError_t launch_levels_scan(const double* d, int64_t n, int cx, double* scratch, unsigned* counter, double* out,
                               cudaStream_t st);
cudaError_t launch_levels_partner(const double* d, int64_t n, int cx, int64_t row, double thresh,
                                  unsigned long long* first, cudaStream_t st);
cudaError_t launch_rowptr_uniform(const int64_t* rp, int64_t n, int64_t per, unsigned* bad, cudaStream_t st);
int levels_scratch_doubles();
cudaError_t launch_unit(const double* z, double* out, int64_t n, double* scratch /*[297]*/, unsigned* counter,
                        cudaStream_t st);
cudaError_t launch_rowdot(const DevSolve& s, const double* delta, const DevCsr* csr, cudaStream_t st);
cudaError_t launch_set_diag_delta(const DevSolve& s, const double* delta, const DevCsr* csr,
                                  cudaStream_t st);

}  // namespace dpt
