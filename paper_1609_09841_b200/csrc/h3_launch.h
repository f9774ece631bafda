// Internal launcher declarations shared by the CUDA translation units and the
// C-ABI layer (h3_capi.cu).  Not part of the public ABI (see include/h3b200.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "h3_common.cuh"

namespace h3 {

// Grid geometry of one launch.  Cells [z_begin, z_end) along x3 are processed;
// x1/x2 are always periodic.  Along x3 node planes wrap modulo M3 when
// periodic_z != 0, otherwise planes -1 and M3 are ghost planes stored
// contiguously before/after the field (slab decomposition).
struct Dims {
    int64_t M1, M2, M3;
    int64_t z_begin, z_end;
    int periodic_z;
    // periodic_z == 0 only: where the ghost planes -1 and M3 live when they are not stored next
    // to the field (h3_fused_pass_halo: the neighbour's boundary plane, read in place over
    // NVLink through a CUDA-IPC mapping); nullptr = contiguous with the field
    const double* ghost_lo = nullptr;
    const double* ghost_hi = nullptr;
    // column-band width of the tile rasterisation (band_tile below; 0 = plain row order), set by
    // the launchers of the tile-march kernels
    int band = 0;
};

// Base of node plane gz of a (slab) field: the field itself, or a separately held ghost plane.
__device__ __forceinline__ const double* plane_base(const double* src, int64_t gz, int64_t plane_elems,
                                                    const Dims& d) {
    if (d.ghost_lo != nullptr && gz < 0) return d.ghost_lo;
    if (d.ghost_hi != nullptr && gz >= d.M3) return d.ghost_hi;
    return src + gz * plane_elems;
}

// Literal (bit-faithful) operator bundle: exactly the reference's factor arrays
// (pipeline.py:197-207), carried as kernel parameters (constant bank).
template <typename T, int N>
struct LitOps {
    static constexpr int S = 2 * N + 2;
    T H[S * S];
    T f1[S], f2[S], f3[S];
    T cf[H3_MAX_STAGES];
    int q;
};

// Separable operator bundle: per-axis node-to-node maps A_k = S_k[0:n, :] H
// (n x 2n, [axis][m][a*n + j]) and the shift rows S_k[0:n, :] (n x s).
template <int N>
struct SepOps {
    static constexpr int n = N + 1, S = 2 * N + 2;
    double A[3][n][S];
    double Sh[3][n][S];
};

// Host operator math (h3_capi.cu): fills A and S from the reference's own
// arguments (N, H, delta = cfac[0], 1/h_k = fac_k[0]) in extended precision.
void build_separable(int order_n, const double* h_mat, const double* fac1, const double* fac2,
                     const double* fac3, double delta, double* A /*3*n*s*/, double* Sh /*3*n*s*/);

// ---- launchers (return cudaError_t as int) --------------------------------
template <typename T>
int literal_launch(int mode /*0 fused,1 recon,2 evolve*/, bool fast, const T* in, T* out,
                   const Dims& d, int order_n, const T* H, const T* f1, const T* f2,
                   const T* f3, const T* cf, int q, int off, cudaStream_t st,
                   unsigned long long* first_bad, const unsigned long long* guard);

int sep_fused_launch(const double* src, double* dst, const Dims& d, int order_n,
                     const double* A, int off, cudaStream_t st, unsigned long long* first_bad,
                     const unsigned long long* guard);
int sep_fused_dmma3_launch(const double* src, double* dst, const Dims& d, const double* A, int off,
                           cudaStream_t st, unsigned long long* first_bad,
                           const unsigned long long* guard);
int sep_fused_dmma3_ws_launch(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                              cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                              int variant);
int sep_fused_dmma3x_launch(const double* src, double* dst, const Dims& d, const SepOps<3>& ops, int off,
                            cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                            int variant);
int sep_fused_dmma5_launch(const double* src, double* dst, const Dims& d, const double* A, int off,
                           cudaStream_t st, unsigned long long* first_bad,
                           const unsigned long long* guard);
int sep_fused_dmma5_ws_launch(const double* src, double* dst, const Dims& d, const double* A, int off,
                              cudaStream_t st, unsigned long long* first_bad, const unsigned long long* guard,
                              int variant);
int recon_dmma5_launch(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                       cudaStream_t st, const unsigned long long* guard);
int recon_dmma5_ws_launch(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                          cudaStream_t st, const unsigned long long* guard, int variant);
int recon_dmma3_launch(const double* src, double* coeff, const Dims& d, const double* h_mat, int off,
                       cudaStream_t st, const unsigned long long* guard);
int recon_sep_launch(const double* src, double* coeff, const Dims& d, int order_n, const double* h_mat,
                     int off, cudaStream_t st, const unsigned long long* guard);
int sep_evolve_launch(const double* coeff, double* dst, const Dims& d, int order_n,
                      const double* Sh, cudaStream_t st, unsigned long long* first_bad,
                      const unsigned long long* guard);

int init_separable_launch(double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n,
                          int nterms, const double* t1, const double* t2, const double* t3,
                          cudaStream_t st);
int error_norms_launch(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                       int nterms, const double* e1, const double* e2, const double* e3,
                       double* d_partials, int64_t n_partials, double* d_out, cudaStream_t st);
int check_finite_launch(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                        unsigned long long* first_bad, cudaStream_t st);

int num_sms();

// Band width a launcher uses: its compiled default, or (tools library only) H3_BAND.
int band_width(int dflt);

// Tile rasterisation.  The hardware starts CTAs in linear block order (x fastest), so with a plain
// mapping the CTAs resident at one time cover ~148 / gx full tile rows: every tile on the lower
// edge of that strip re-reads its halo node row from DRAM when the next strip runs (the row was
// evicted long before).  `band_tile` walks the tile grid in column bands of `band` tiles instead
// (row-major inside a band), so the resident CTAs cover a compact block whose perimeter -- the
// only halo that misses L2 -- is ~3x shorter.  Clusters of `cy` CTAs along y keep their pairing:
// the unit remapped is the cluster (x, y / cy); band = 0 is the identity.
__device__ __forceinline__ void band_tile(int band, int cy, int& bx, int& by) {
    bx = (int)blockIdx.x;
    by = (int)blockIdx.y;
    if (band <= 0) return;
    const int gx = (int)gridDim.x, gu = (int)gridDim.y / cy;
    const int lin = bx + gx * (by / cy);
    const int b = lin / (band * gu), r = lin - b * (band * gu);
    const int w = min(band, gx - b * band);  // width of this band (the last one may be narrower)
    const int uy = r / w;
    bx = b * band + (r - uy * w);
    by = uy * cy + (int)blockIdx.y % cy;
}

// z-chunk length for a tile march over nz cell planes with `tiles` x1-x2 tiles and `slots`
// resident CTAs: minimises waves x (planes per CTA + halo plane + ~2 planes of pipeline fill),
// waves = ceil(tiles * chunks / slots), over chunk lengths >= min_chunk.  (At 512^3 m=3 this is
// one chunk per tile -- 4736 tiles = 32 full waves; at 128^3 it avoids a 10 %-full last wave.)
inline int64_t choose_zchunk(int64_t tiles, int64_t nz, int64_t slots, int64_t min_chunk = 8) {
    if (nz <= min_chunk) return nz > 0 ? nz : 1;
    if (slots < 1) slots = 1;
    int64_t best = nz;
    double best_cost = 1e300;
    for (int64_t zs = 1;; ++zs) {
        const int64_t zc = (nz + zs - 1) / zs;
        if (zc < min_chunk) break;
        const int64_t chunks = (nz + zc - 1) / zc;
        const int64_t waves = (tiles * chunks + slots - 1) / slots;
        const double cost = (double)waves * (double)(zc + 3);
        if (cost < best_cost * (1.0 - 1e-9)) {
            best_cost = cost;
            best = zc;
        }
        if (zc == min_chunk) break;
    }
    return best;
}

}  // namespace h3
