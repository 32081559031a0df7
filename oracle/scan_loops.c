/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by, or called
 * from the product path (paper_2602_08810_b200/).  Only tests/, the smoke
 * check in __graft_entry__.py and bench.py's cpu_baseline / --impl reference
 * leg may load the shared object built from this file.
 *
 * Plain-C restatement of the ten native loops of the reference's scan
 * operator, reference file pkg/src/linrec/_scan_kernels.py:
 *
 *   scan_const        :17-26    out[k] = a*out[k-1] + b[k], x0 seed
 *   scan_var          :29-37    same with a[k]
 *   compose_const     :40-57    fold a block into (acc_a, acc_b)
 *   compose_var       :60-71
 *   local_scan_const  :74-87    zero-init chunk scan + total a-product
 *   local_scan_var    :90-102
 *   fixup_const       :105-116  out[k] += a^{k+1} * xin
 *   fixup_var         :119-128  out[k] += (prod_{j<=k} a_j) * xin
 *   backward_const    :131-141  out[k] = gx[k] + aconj*out[k+1]
 *   backward_var      :144-153  out[k] = gx[k] + aconj[k+1]*out[k+1]
 *
 * Same contract as the reference: time-major [L, N] C-contiguous arrays,
 * caller-allocated outputs, no conjugation inside (callers pass conj(a)),
 * L >= 1 (callers enforce).  The loop order (lane-outer, time-inner) and the
 * operation order inside each step are kept identical so that float results
 * match the numba kernels bit-for-bit under strict IEEE evaluation (compiled
 * with -O2 -fno-fast-math -ffp-contract=off).  The four dtypes of the
 * reference (float32/64, complex64/128) are generated from one macro.
 *
 * The functions hold no global state and are reentrant, mirroring numba's
 * nogil kernels: ctypes releases the GIL around each call, so a Python thread
 * pool over disjoint chunks runs them truly in parallel, exactly like the
 * reference's ThreadPoolExecutor over nogil kernels (scan.py:46-55).
 */
#include <complex.h>
#include <stdint.h>

#define DEFINE_LOOPS(SUF, T)                                                   \
void scan_const_##SUF(const T *a, const T *b, const T *x0, T *out,            \
                      int64_t L, int64_t N) {                                  \
    for (int64_t j = 0; j < N; ++j) {                                          \
        T x = x0[j];                                                           \
        const T aj = a[j];                                                     \
        for (int64_t k = 0; k < L; ++k) {                                      \
            x = aj * x + b[k * N + j];                                         \
            out[k * N + j] = x;                                                \
        }                                                                      \
    }                                                                          \
}                                                                              \
void scan_var_##SUF(const T *a, const T *b, const T *x0, T *out,              \
                    int64_t L, int64_t N) {                                    \
    for (int64_t j = 0; j < N; ++j) {                                          \
        T x = x0[j];                                                           \
        for (int64_t k = 0; k < L; ++k) {                                      \
            x = a[k * N + j] * x + b[k * N + j];                               \
            out[k * N + j] = x;                                                \
        }                                                                      \
    }                                                                          \
}                                                                              \
void compose_const_##SUF(const T *a, const T *b, T *acc_a, T *acc_b,          \
                         int64_t L, int64_t N) {                               \
    for (int64_t j = 0; j < N; ++j) {                                          \
        const T aj = a[j];                                                     \
        T xa = acc_a[j], xb = acc_b[j];                                        \
        for (int64_t k = 0; k < L; ++k) {                                      \
            xb = aj * xb + b[k * N + j];                                       \
            xa = aj * xa;                                                      \
        }                                                                      \
        acc_a[j] = xa;                                                         \
        acc_b[j] = xb;                                                         \
    }                                                                          \
}                                                                              \
void compose_var_##SUF(const T *a, const T *b, T *acc_a, T *acc_b,            \
                       int64_t L, int64_t N) {                                 \
    for (int64_t j = 0; j < N; ++j) {                                          \
        T xa = acc_a[j], xb = acc_b[j];                                        \
        for (int64_t k = 0; k < L; ++k) {                                      \
            const T ak = a[k * N + j];                                         \
            xb = ak * xb + b[k * N + j];                                       \
            xa = ak * xa;                                                      \
        }                                                                      \
        acc_a[j] = xa;                                                         \
        acc_b[j] = xb;                                                         \
    }                                                                          \
}                                                                              \
void local_scan_const_##SUF(const T *a, const T *b, T *out, T *prod,          \
                            int64_t L, int64_t N) {                            \
    for (int64_t j = 0; j < N; ++j) {                                          \
        const T aj = a[j];                                                     \
        T x = b[j];                                                            \
        out[j] = x;                                                            \
        T p = aj;                                                              \
        for (int64_t k = 1; k < L; ++k) {                                      \
            x = aj * x + b[k * N + j];                                         \
            out[k * N + j] = x;                                                \
            p = p * aj;                                                        \
        }                                                                      \
        prod[j] = p;                                                           \
    }                                                                          \
}                                                                              \
void local_scan_var_##SUF(const T *a, const T *b, T *out, T *prod,            \
                          int64_t L, int64_t N) {                              \
    for (int64_t j = 0; j < N; ++j) {                                          \
        T x = b[j];                                                            \
        out[j] = x;                                                            \
        T p = a[j];                                                            \
        for (int64_t k = 1; k < L; ++k) {                                      \
            const T ak = a[k * N + j];                                         \
            x = ak * x + b[k * N + j];                                         \
            out[k * N + j] = x;                                                \
            p = p * ak;                                                        \
        }                                                                      \
        prod[j] = p;                                                           \
    }                                                                          \
}                                                                              \
void fixup_const_##SUF(const T *a, const T *xin, T *out,                      \
                       int64_t L, int64_t N) {                                 \
    for (int64_t j = 0; j < N; ++j) {                                          \
        const T aj = a[j], v = xin[j];                                         \
        T p = aj;                                                              \
        out[j] = out[j] + p * v;                                               \
        for (int64_t k = 1; k < L; ++k) {                                      \
            p = p * aj;                                                        \
            out[k * N + j] = out[k * N + j] + p * v;                           \
        }                                                                      \
    }                                                                          \
}                                                                              \
void fixup_var_##SUF(const T *a, const T *xin, T *out,                        \
                     int64_t L, int64_t N) {                                   \
    for (int64_t j = 0; j < N; ++j) {                                          \
        const T v = xin[j];                                                    \
        T p = a[j];                                                            \
        out[j] = out[j] + p * v;                                               \
        for (int64_t k = 1; k < L; ++k) {                                      \
            p = p * a[k * N + j];                                              \
            out[k * N + j] = out[k * N + j] + p * v;                           \
        }                                                                      \
    }                                                                          \
}                                                                              \
void backward_const_##SUF(const T *aconj, const T *gx, T *out,                \
                          int64_t L, int64_t N) {                              \
    for (int64_t j = 0; j < N; ++j) {                                          \
        const T aj = aconj[j];                                                 \
        T g = gx[(L - 1) * N + j];                                             \
        out[(L - 1) * N + j] = g;                                              \
        for (int64_t k = L - 2; k >= 0; --k) {                                 \
            g = gx[k * N + j] + aj * g;                                        \
            out[k * N + j] = g;                                                \
        }                                                                      \
    }                                                                          \
}                                                                              \
void backward_var_##SUF(const T *aconj, const T *gx, T *out,                  \
                        int64_t L, int64_t N) {                                \
    for (int64_t j = 0; j < N; ++j) {                                          \
        T g = gx[(L - 1) * N + j];                                             \
        out[(L - 1) * N + j] = g;                                              \
        for (int64_t k = L - 2; k >= 0; --k) {                                 \
            g = gx[k * N + j] + aconj[(k + 1) * N + j] * g;                    \
            out[k * N + j] = g;                                                \
        }                                                                      \
    }                                                                          \
}

DEFINE_LOOPS(f32, float)
DEFINE_LOOPS(f64, double)
DEFINE_LOOPS(c64, float _Complex)
DEFINE_LOOPS(c128, double _Complex)
