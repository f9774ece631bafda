// C ABI (include/h3b200.h): argument validation, variant selection and the
// host-side separable operator math.  Everything here is plain C++; the
// kernels live in h3_literal.cu, h3_separable.cu and h3_problems.cu.
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../../include/h3b200.h"
#include "h3_launch.h"

#define H3_VERSION_STRING "h3b200 0.1.0 (sm_100a)"

namespace h3 {

void build_separable(int order_n, const double* h_mat, const double* fac1, const double* fac2,
                     const double* fac3, double delta, double* A, double* Sh) {
    const int n = order_n + 1, s = 2 * n;
    const double* facs[3] = {fac1, fac2, fac3};
    for (int k = 0; k < 3; ++k) {
        // delta / h_k from the reference's own arguments: fac_k[0] = 1 * (1/h_k)
        const long double r = (long double)delta * (long double)facs[k][0];
        long double S[H3_MAX_ORDER + 1][2 * H3_MAX_ORDER + 2];
        for (int m = 0; m < n; ++m)
            for (int j = 0; j < s; ++j) {
                if (j < m) { S[m][j] = 0.0L; continue; }
                long double binom = 1.0L;  // C(j, m)
                for (int t = 1; t <= j - m; ++t) binom = binom * (long double)(m + t) / (long double)t;
                long double pw = 1.0L;
                for (int t = 0; t < j - m; ++t) pw *= r;
                S[m][j] = binom * pw;
            }
        for (int m = 0; m < n; ++m)
            for (int c = 0; c < s; ++c) {
                if (Sh) Sh[(k * n + m) * s + c] = (double)S[m][c];
                if (A) {
                    long double acc = 0.0L;
                    for (int j = 0; j < s; ++j) acc += S[m][j] * (long double)h_mat[j * s + c];
                    A[(k * n + m) * s + c] = (double)acc;
                }
            }
    }
}

}  // namespace h3

using h3::Dims;

static int check_common(int64_t M1, int64_t M2, int64_t M3, int order_n, int64_t z_begin,
                        int64_t z_end) {
    if (order_n < 0 || order_n > H3_MAX_ORDER) return H3_ERR_ORDER;
    if (M1 < 1 || M2 < 1 || M3 < 1) return H3_ERR_ARG;
    if (M1 > (1ll << 30) || M2 > (1ll << 30)) return H3_ERR_ARG;
    if (z_begin < 0 || z_end > M3 || z_begin > z_end) return H3_ERR_ARG;
    return 0;
}

static int exact_stages(int order_n) { return 3 * (2 * order_n + 1); }

template <typename T>
static int fused_impl(const T* src, T* dst, int64_t M1, int64_t M2, int64_t M3, int order_n,
                      const T* h_mat, const T* fac1, const T* fac2, const T* fac3, const T* cfac,
                      int q, int off, int64_t z_begin, int64_t z_end, int periodic_z, int variant,
                      void* stream, unsigned long long* d_first_bad,
                      const unsigned long long* d_guard) {
    int rc = check_common(M1, M2, M3, order_n, z_begin, z_end);
    if (rc) return rc;
    if (!src || !dst || !h_mat || !fac1 || !fac2 || !fac3 || !cfac) return H3_ERR_ARG;
    if (off != 0 && off != -1) return H3_ERR_ARG;
    if (q < 1) return H3_ERR_STAGES;
    Dims d{M1, M2, M3, z_begin, z_end, periodic_z ? 1 : 0};
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    bool separable;
    switch (variant) {
        case H3_VARIANT_AUTO: separable = sizeof(T) == 8 && q >= exact_stages(order_n); break;
        case H3_VARIANT_LITERAL: separable = false; break;
        case H3_VARIANT_SEPARABLE:
            if (sizeof(T) != 8) return H3_ERR_VARIANT;
            if (q < exact_stages(order_n)) return H3_ERR_STAGES;
            separable = true;
            break;
        default: return H3_ERR_VARIANT;
    }
    if (separable) {
        const int n = order_n + 1, s = 2 * n;
        double A[3 * (H3_MAX_ORDER + 1) * (2 * H3_MAX_ORDER + 2)];
        h3::build_separable(order_n, (const double*)h_mat, (const double*)fac1, (const double*)fac2,
                            (const double*)fac3, (double)cfac[0], A, nullptr);
        (void)s;
        return h3::sep_fused_launch((const double*)src, (double*)dst, d, order_n, A, off, st,
                                    d_first_bad, d_guard);
    }
    // the literal kernels keep the q stage factors in a fixed-size parameter block; the
    // separable path uses cfac[0] only, so the cap applies here alone
    if (q > H3_MAX_STAGES) return H3_ERR_STAGES;
    return h3::literal_launch<T>(0, false, src, dst, d, order_n, h_mat, fac1, fac2, fac3, cfac, q,
                                 off, st, d_first_bad, d_guard);
}

template <typename T>
static int recon_impl(const T* src, T* coeff, int64_t M1, int64_t M2, int64_t M3, int order_n,
                      const T* h_mat, int off, int64_t z_begin, int64_t z_end, int periodic_z,
                      int variant, void* stream, const unsigned long long* d_guard) {
    int rc = check_common(M1, M2, M3, order_n, z_begin, z_end);
    if (rc) return rc;
    if (!src || !coeff || !h_mat) return H3_ERR_ARG;
    if (off != 0 && off != -1) return H3_ERR_ARG;
    bool fast;
    switch (variant) {
        case H3_VARIANT_AUTO: fast = sizeof(T) == 8; break;
        case H3_VARIANT_LITERAL: fast = false; break;
        case H3_VARIANT_SEPARABLE:
            if (sizeof(T) != 8) return H3_ERR_VARIANT;
            fast = true;
            break;
        default: return H3_ERR_VARIANT;
    }
    Dims d{M1, M2, M3, z_begin, z_end, periodic_z ? 1 : 0};
    if (fast && sizeof(T) == 8) {
        // node-factorised reconstruction: FP64 tensor cores at N = 3 and 5, DFMA otherwise
#ifdef H3_MEASURE
        // tools library only (H3_RECON_IMPL=sep: DFMA kernel at N = 3 too; =fma: per-cell sweeps)
        static const int impl = [] {
            const char* e = getenv("H3_RECON_IMPL");
            if (e && strcmp(e, "fma") == 0) return 2;
            if (e && strcmp(e, "sep") == 0) return 1;
            return 0;
        }();
#else
        constexpr int impl = 0;
#endif
        cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
        if (impl == 0 && order_n == 3)
            return h3::recon_dmma3_launch((const double*)src, (double*)coeff, d, (const double*)h_mat, off, st,
                                          d_guard);
        if (impl == 0 && order_n == 5)
            return h3::recon_dmma5_launch((const double*)src, (double*)coeff, d, (const double*)h_mat, off, st,
                                          d_guard);
        if (impl != 2)
            return h3::recon_sep_launch((const double*)src, (double*)coeff, d, order_n, (const double*)h_mat, off,
                                        st, d_guard);
    }
    return h3::literal_launch<T>(1, fast, src, coeff, d, order_n, h_mat, nullptr, nullptr, nullptr,
                                 nullptr, 1, off, reinterpret_cast<cudaStream_t>(stream), nullptr,
                                 d_guard);
}

template <typename T>
static int evolve_impl(const T* coeff, T* dst, int64_t M1, int64_t M2, int64_t M3, int order_n,
                       const T* fac1, const T* fac2, const T* fac3, const T* cfac, int q,
                       int64_t z_begin, int64_t z_end, int variant, void* stream,
                       unsigned long long* d_first_bad, const unsigned long long* d_guard) {
    int rc = check_common(M1, M2, M3, order_n, z_begin, z_end);
    if (rc) return rc;
    if (!coeff || !dst || !fac1 || !fac2 || !fac3 || !cfac) return H3_ERR_ARG;
    if (q < 1) return H3_ERR_STAGES;
    bool separable;
    switch (variant) {
        case H3_VARIANT_AUTO: separable = sizeof(T) == 8 && q >= exact_stages(order_n); break;
        case H3_VARIANT_LITERAL: separable = false; break;
        case H3_VARIANT_SEPARABLE:
            if (sizeof(T) != 8) return H3_ERR_VARIANT;
            if (q < exact_stages(order_n)) return H3_ERR_STAGES;
            separable = true;
            break;
        default: return H3_ERR_VARIANT;
    }
    Dims d{M1, M2, M3, z_begin, z_end, 1};
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    if (separable) {
        const int n = order_n + 1, s = 2 * n;
        double Sh[3 * (H3_MAX_ORDER + 1) * (2 * H3_MAX_ORDER + 2)];
        double hid[(2 * H3_MAX_ORDER + 2) * (2 * H3_MAX_ORDER + 2)];
        memset(hid, 0, sizeof(hid));
        for (int i = 0; i < s; ++i) hid[i * s + i] = 1.0;
        h3::build_separable(order_n, hid, (const double*)fac1, (const double*)fac2,
                            (const double*)fac3, (double)cfac[0], nullptr, Sh);
        return h3::sep_evolve_launch((const double*)coeff, (double*)dst, d, order_n, Sh, st,
                                     d_first_bad, d_guard);
    }
    if (q > H3_MAX_STAGES) return H3_ERR_STAGES;  // literal only (see fused_impl)
    return h3::literal_launch<T>(2, false, coeff, dst, d, order_n, nullptr, fac1, fac2, fac3, cfac,
                                 q, 0, st, d_first_bad, d_guard);
}

// Fused half step of a slab whose ghost planes are held elsewhere (peer GPU memory).
static int fused_halo_impl(const double* src, double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n,
                           const double* h_mat, const double* fac1, const double* fac2, const double* fac3,
                           const double* cfac, int q, int off, int64_t z_begin, int64_t z_end,
                           const double* ghost_lo, const double* ghost_hi, int variant, void* stream,
                           unsigned long long* d_first_bad, const unsigned long long* d_guard) {
    int rc = check_common(M1, M2, M3, order_n, z_begin, z_end);
    if (rc) return rc;
    if (!src || !dst || !h_mat || !fac1 || !fac2 || !fac3 || !cfac) return H3_ERR_ARG;
    if (off != 0 && off != -1) return H3_ERR_ARG;
    if (off == 0 && z_end == M3 && !ghost_hi) return H3_ERR_ARG;   // cell M3-1 reads plane M3
    if (off == -1 && z_begin == 0 && !ghost_lo) return H3_ERR_ARG;  // cell 0 reads plane -1
    if (q < exact_stages(order_n)) return H3_ERR_STAGES;
    // the tile-march kernels with TMA plane loads take the ghost pointers (N = 3, 5)
    if ((variant != H3_VARIANT_AUTO && variant != H3_VARIANT_SEPARABLE) || (order_n != 3 && order_n != 5))
        return H3_ERR_VARIANT;
    Dims d{M1, M2, M3, z_begin, z_end, 0};
    d.ghost_lo = ghost_lo;
    d.ghost_hi = ghost_hi;
    const int n = order_n + 1, s = 2 * n;
    double A[3 * (H3_MAX_ORDER + 1) * (2 * H3_MAX_ORDER + 2)];
    h3::build_separable(order_n, h_mat, fac1, fac2, fac3, cfac[0], A, nullptr);
    (void)s;
    (void)n;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    return order_n == 3 ? h3::sep_fused_dmma3_launch(src, dst, d, A, off, st, d_first_bad, d_guard)
                        : h3::sep_fused_dmma5_launch(src, dst, d, A, off, st, d_first_bad, d_guard);
}

extern "C" {

int h3_fused_pass_halo(const double* src, double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n,
                       const double* h_mat, const double* fac1, const double* fac2, const double* fac3,
                       const double* cfac, int q, int off, int64_t z_begin, int64_t z_end,
                       const double* ghost_lo, const double* ghost_hi, int variant, void* stream,
                       unsigned long long* d_first_bad, const unsigned long long* d_guard) {
    return fused_halo_impl(src, dst, M1, M2, M3, order_n, h_mat, fac1, fac2, fac3, cfac, q, off, z_begin,
                           z_end, ghost_lo, ghost_hi, variant, stream, d_first_bad, d_guard);
}

// CUDA IPC of a device buffer that may sit inside a larger allocation (torch's caching
// allocator): export the handle of the containing allocation plus the byte offset.
typedef int (*h3_cuMemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);

int h3_ipc_export(const void* ptr, unsigned char* handle64, int64_t* offset) {
    if (!ptr || !handle64 || !offset) return H3_ERR_ARG;
    static h3_cuMemGetAddressRange_t range = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (h3_cuMemGetAddressRange_t) nullptr;
        return (h3_cuMemGetAddressRange_t)fn;
    }();
    if (!range) return (int)cudaErrorNotSupported;
    unsigned long long base = 0;
    size_t size = 0;
    if (range(&base, &size, (unsigned long long)(uintptr_t)ptr) != 0) return (int)cudaErrorInvalidDevicePointer;
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base);
    if (e != cudaSuccess) return (int)e;
    memcpy(handle64, &h, sizeof(h));
    *offset = (int64_t)((uintptr_t)ptr - (uintptr_t)base);
    return 0;
}

int h3_ipc_open(const unsigned char* handle64, void** base_out) {
    if (!handle64 || !base_out) return H3_ERR_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    return (int)cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
}

int h3_ipc_close(void* base) { return base ? (int)cudaIpcCloseMemHandle(base) : H3_ERR_ARG; }

int h3_fused_pass(const double* src, double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n,
                  const double* h_mat, const double* fac1, const double* fac2, const double* fac3,
                  const double* cfac, int q, int off, int64_t z_begin, int64_t z_end,
                  int periodic_z, int variant, void* stream, unsigned long long* d_first_bad,
                  const unsigned long long* d_guard) {
    return fused_impl<double>(src, dst, M1, M2, M3, order_n, h_mat, fac1, fac2, fac3, cfac, q, off,
                              z_begin, z_end, periodic_z, variant, stream, d_first_bad, d_guard);
}

int h3_fused_pass_f32(const float* src, float* dst, int64_t M1, int64_t M2, int64_t M3,
                      int order_n, const float* h_mat, const float* fac1, const float* fac2,
                      const float* fac3, const float* cfac, int q, int off, int64_t z_begin,
                      int64_t z_end, int periodic_z, int variant, void* stream,
                      unsigned long long* d_first_bad, const unsigned long long* d_guard) {
    return fused_impl<float>(src, dst, M1, M2, M3, order_n, h_mat, fac1, fac2, fac3, cfac, q, off,
                             z_begin, z_end, periodic_z, variant, stream, d_first_bad, d_guard);
}

int h3_recon_pass(const double* src, double* coeff, int64_t M1, int64_t M2, int64_t M3,
                  int order_n, const double* h_mat, int off, int64_t z_begin, int64_t z_end,
                  int periodic_z, int variant, void* stream, const unsigned long long* d_guard) {
    return recon_impl<double>(src, coeff, M1, M2, M3, order_n, h_mat, off, z_begin, z_end,
                              periodic_z, variant, stream, d_guard);
}

int h3_recon_pass_f32(const float* src, float* coeff, int64_t M1, int64_t M2, int64_t M3,
                      int order_n, const float* h_mat, int off, int64_t z_begin, int64_t z_end,
                      int periodic_z, int variant, void* stream, const unsigned long long* d_guard) {
    return recon_impl<float>(src, coeff, M1, M2, M3, order_n, h_mat, off, z_begin, z_end,
                             periodic_z, variant, stream, d_guard);
}

int h3_evolve_pass(const double* coeff, double* dst, int64_t M1, int64_t M2, int64_t M3,
                   int order_n, const double* fac1, const double* fac2, const double* fac3,
                   const double* cfac, int q, int64_t z_begin, int64_t z_end, int variant,
                   void* stream, unsigned long long* d_first_bad,
                   const unsigned long long* d_guard) {
    return evolve_impl<double>(coeff, dst, M1, M2, M3, order_n, fac1, fac2, fac3, cfac, q, z_begin,
                               z_end, variant, stream, d_first_bad, d_guard);
}

int h3_evolve_pass_f32(const float* coeff, float* dst, int64_t M1, int64_t M2, int64_t M3,
                       int order_n, const float* fac1, const float* fac2, const float* fac3,
                       const float* cfac, int q, int64_t z_begin, int64_t z_end, int variant,
                       void* stream, unsigned long long* d_first_bad,
                       const unsigned long long* d_guard) {
    return evolve_impl<float>(coeff, dst, M1, M2, M3, order_n, fac1, fac2, fac3, cfac, q, z_begin,
                              z_end, variant, stream, d_first_bad, d_guard);
}

int h3_separable_operators(int order_n, const double* h_mat, const double* fac1,
                           const double* fac2, const double* fac3, const double* cfac, int q,
                           double* A_out, double* S_out) {
    if (order_n < 0 || order_n > H3_MAX_ORDER) return H3_ERR_ORDER;
    if (!h_mat || !fac1 || !fac2 || !fac3 || !cfac) return H3_ERR_ARG;
    if (q < 1) return H3_ERR_STAGES;
    h3::build_separable(order_n, h_mat, fac1, fac2, fac3, cfac[0], A_out, S_out);
    return 0;
}

int h3_init_separable(double* dst, int64_t M1, int64_t M2, int64_t M3, int order_n, int nterms,
                      const double* t1, const double* t2, const double* t3, void* stream) {
    int rc = check_common(M1, M2, M3, order_n, 0, M3);
    if (rc) return rc;
    if (!dst || !t1 || !t2 || !t3 || nterms < 1) return H3_ERR_ARG;
    return h3::init_separable_launch(dst, M1, M2, M3, order_n, nterms, t1, t2, t3,
                                     reinterpret_cast<cudaStream_t>(stream));
}

int h3_error_norms(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                   int nterms, const double* e1, const double* e2, const double* e3,
                   double* d_partials, int64_t n_partials, double* d_out, void* stream) {
    int rc = check_common(M1, M2, M3, order_n, 0, M3);
    if (rc) return rc;
    if (!field || !e1 || !e2 || !e3 || !d_partials || !d_out || nterms < 1 || n_partials < 1)
        return H3_ERR_ARG;
    return h3::error_norms_launch(field, M1, M2, M3, order_n, nterms, e1, e2, e3, d_partials,
                                  n_partials, d_out, reinterpret_cast<cudaStream_t>(stream));
}

int h3_check_finite(const double* field, int64_t M1, int64_t M2, int64_t M3, int order_n,
                    unsigned long long* d_first_bad, void* stream) {
    int rc = check_common(M1, M2, M3, order_n, 0, M3);
    if (rc) return rc;
    if (!field || !d_first_bad) return H3_ERR_ARG;
    return h3::check_finite_launch(field, M1, M2, M3, order_n, d_first_bad,
                                   reinterpret_cast<cudaStream_t>(stream));
}

const char* h3_version(void) { return H3_VERSION_STRING; }

const char* h3_error_string(int status) {
    switch (status) {
        case 0: return "success";
        case H3_ERR_ARG: return "invalid argument (pointer, size, offset or slab range)";
        case H3_ERR_ORDER: return "order_n outside the supported range";
        case H3_ERR_STAGES: return "stage count outside the supported range for this variant";
        case H3_ERR_VARIANT: return "variant not available for this precision/kernel";
    }
    if (status > 0) return cudaGetErrorString((cudaError_t)status);
    return "unknown h3b200 status";
}

int h3_max_order(void) { return H3_MAX_ORDER; }
int h3_max_stages(void) { return H3_MAX_STAGES; }

}  // extern "C"
