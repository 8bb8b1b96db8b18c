// oracle/_ref driver: a C-ABI over the UNMODIFIED reference solvers, compiled from
// the headers where they lie under /root/reference/proj/core/include (recipe:
// oracle/ref/Makefile). TEST INFRASTRUCTURE ONLY: loaded by tests/ and by
// bench.py's reference / cpu_baseline arm, never by the product library.
//
// Matrices cross this boundary in "slot order": the reference's own internal
// storage order of BlockBandedMatrix (block_banded.hpp:58-60), i.e. slot
// a*(2w+1) + off + w, each slot bs x bs complex128 column-major (interleaved
// re,im), the (rows(a) x cols(a+off)) block in its top-left corner with ld = bs.
// Out-of-band slots are ignored on input and zero on output.
#include <cstdint>
#include <cstring>
#include <string>

#include "bbsi/cost_model.hpp"
#include "bbsi/ddrgf.hpp"
#include "bbsi/io.hpp"
#include "bbsi/rgf.hpp"
#include "bbsi/threading.hpp"
#include "helpers.hpp"  // reference tests/helpers.hpp: random_hermitian

using namespace bbsi;
using cd = std::complex<double>;

namespace {

thread_local std::string g_err;

BlockLayout layout_of(int l, int w, int bs, const int* sizes) {
    std::vector<int> s(l);
    for (int a = 0; a < l; ++a) s[a] = sizes ? sizes[a] : bs;
    return BlockLayout(l, s, w);
}

size_t slot_elems(int bs) { return size_t(bs) * bs; }

BlockBandedMatrix<cd> from_slots(const BlockLayout& lay, int bs, const double* p) {
    BlockBandedMatrix<cd> m(lay);
    const int w = lay.bandwidth;
    const cd* src = reinterpret_cast<const cd*>(p);
    for (int a = 0; a < lay.num_layers; ++a)
        for (int off = -w; off <= w; ++off) {
            if (!m.in_band(a, off)) continue;
            auto& blk = m.block(a, off);
            const cd* s = src + (size_t(a) * (2 * w + 1) + off + w) * slot_elems(bs);
            for (int j = 0; j < blk.cols(); ++j)
                for (int i = 0; i < blk.rows(); ++i) blk(i, j) = s[size_t(j) * bs + i];
        }
    return m;
}

void to_slots(const BlockBandedMatrix<cd>& m, int bs, double* p) {
    const int w = m.bandwidth();
    const int l = m.num_layers();
    cd* dst = reinterpret_cast<cd*>(p);
    std::memset(p, 0, sizeof(cd) * size_t(l) * (2 * w + 1) * slot_elems(bs));
    for (int a = 0; a < l; ++a)
        for (int off = -w; off <= w; ++off) {
            if (!m.in_band(a, off)) continue;
            const auto& blk = m.block(a, off);
            cd* d = dst + (size_t(a) * (2 * w + 1) + off + w) * slot_elems(bs);
            for (int j = 0; j < blk.cols(); ++j)
                for (int i = 0; i < blk.rows(); ++i) d[size_t(j) * bs + i] = blk(i, j);
        }
}

void put_counters(const KernelCounters& c, long long* out) {
    if (!out) return;
    out[0] = c.n_gemm;
    out[1] = c.n_lu;
    out[2] = c.n_getrs;
}

template <class F>
int guarded(int* fail_layer, F&& fn) {
    if (fail_layer) *fail_layer = -1;
    try {
        fn();
        return 0;
    } catch (const singular_matrix_error& e) {
        g_err = e.what();
        if (fail_layer) *fail_layer = e.layer();
        return 2;
    } catch (const invalid_argument_error& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 3;
    }
}

void blocks_to(const std::vector<DenseMatrix<cd>>& v, int bs, double* p) {
    if (!p) return;
    cd* dst = reinterpret_cast<cd*>(p);
    std::memset(p, 0, sizeof(cd) * v.size() * slot_elems(bs));
    for (size_t k = 0; k < v.size(); ++k)
        for (int j = 0; j < v[k].cols(); ++j)
            for (int i = 0; i < v[k].rows(); ++i) dst[k * slot_elems(bs) + size_t(j) * bs + i] = v[k](i, j);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_threads(int n) { set_kernel_threads(n); }

int ref_random_spd_like(int l, int w, int bs, const int* sizes, uint64_t seed, double dominance,
                        double* A) {
    return guarded(nullptr, [&] {
        auto m = random_spd_like<cd>(layout_of(l, w, bs, sizes), seed, dominance);
        to_slots(m, bs, A);
    });
}

// .bbm files through the reference's own io.cpp (write_bbm / read_bbm).
int ref_write_bbm(const char* path, int l, int w, int bs, const int* sizes, const double* A) {
    return guarded(nullptr, [&] { write_bbm(path, from_slots(layout_of(l, w, bs, sizes), bs, A)); });
}

// Reads a .bbm file: dims[0..2] = (num_layers, bandwidth, max block size); with A null
// only the dims (and sizes, when non-null and large enough) are filled.
int ref_read_bbm(const char* path, int* dims, int* sizes, int max_layers, double* A) {
    return guarded(nullptr, [&] {
        auto m = read_bbm(path);
        const auto& lay = m.layout();
        int bs = 0;
        for (int b : lay.block_sizes) bs = b > bs ? b : bs;
        dims[0] = lay.num_layers;
        dims[1] = lay.bandwidth;
        dims[2] = bs;
        if (sizes && max_layers >= lay.num_layers)
            for (int a = 0; a < lay.num_layers; ++a) sizes[a] = lay.block_sizes[a];
        if (A) to_slots(m, bs, A);
    });
}

int ref_random_hermitian(int l, int w, int bs, const int* sizes, uint64_t seed, double dominance,
                         double* A) {
    return guarded(nullptr, [&] {
        auto m = testutil::random_hermitian(layout_of(l, w, bs, sizes), seed, dominance);
        to_slots(m, bs, A);
    });
}

int ref_rgf_tridiag(int l, int w, int bs, const int* sizes, const double* A, double* G,
                    long long* counters, int* fail_layer) {
    return guarded(fail_layer, [&] {
        auto lay = layout_of(l, w, bs, sizes);
        auto [g, c] = rgf_tridiag(from_slots(lay, bs, A));
        to_slots(g, bs, G);
        put_counters(c, counters);
    });
}

int ref_rgf_ndiag(int l, int w, int bs, const int* sizes, const double* A, double* G,
                  long long* counters, int* max_update_offset, int* fail_layer) {
    return guarded(fail_layer, [&] {
        auto lay = layout_of(l, w, bs, sizes);
        StructuralTrace trace;
        auto [g, c] = rgf_ndiag(from_slots(lay, bs, A), &trace);
        to_slots(g, bs, G);
        put_counters(c, counters);
        if (max_update_offset) *max_update_offset = trace.max_update_offset;
    });
}

int ref_rgf_fused(int l, int w, int bs, const int* sizes, const double* A, double* G,
                  long long* counters, int* fail_layer) {
    return guarded(fail_layer, [&] {
        auto lay = layout_of(l, w, bs, sizes);
        auto [g, c] = rgf_fused(from_slots(lay, bs, A));
        to_slots(g, bs, G);
        put_counters(c, counters);
    });
}

int ref_rgf_extended(int l, int w, int bs, const int* sizes, const double* A, double* G,
                     double* first_row, double* last_row, double* first_col, double* last_col,
                     long long* counters, int* fail_layer) {
    return guarded(fail_layer, [&] {
        auto lay = layout_of(l, w, bs, sizes);
        auto [ext, c] = rgf_extended(from_slots(lay, bs, A));
        to_slots(ext.core, bs, G);
        blocks_to(ext.first_row, bs, first_row);
        blocks_to(ext.last_row, bs, last_row);
        blocks_to(ext.first_col, bs, first_col);
        blocks_to(ext.last_col, bs, last_col);
        put_counters(c, counters);
    });
}

int ref_ddrgf(int l, int w, int bs, const int* sizes, const double* A, const int* s2_levels,
              int n_levels, int n_threads, int terminal_threads, double* G, long long* counters,
              int* fail_layer) {
    return guarded(fail_layer, [&] {
        auto lay = layout_of(l, w, bs, sizes);
        DomainPlan plan;
        plan.s2_levels.assign(s2_levels, s2_levels + n_levels);
        plan.n_threads = n_threads;
        plan.terminal_threads = terminal_threads;
        auto [g, c] = ddrgf(from_slots(lay, bs, A), plan);
        to_slots(g, bs, G);
        put_counters(c, counters);
    });
}

int ref_oracle_selected_inverse(int l, int w, int bs, const int* sizes, const double* A, double* G) {
    return guarded(nullptr, [&] {
        auto lay = layout_of(l, w, bs, sizes);
        auto g = oracle_selected_inverse(from_slots(lay, bs, A));
        to_slots(g, bs, G);
    });
}

// Reference closed forms (cost_model.hpp:44-61,126-154), exposed so the Python
// restatement of the counters can be pinned against them.
void ref_predict_rgf_counters(long long l, long long* out) { put_counters(predict_rgf_counters(l), out); }
void ref_predict_nrgf_counters(long long l, long long w, long long* out) {
    put_counters(predict_nrgf_counters(l, w), out);
}
int ref_predict_ddrgf_counters(long long l, const int* s2_levels, int n_levels, long long* out) {
    return guarded(nullptr, [&] {
        DomainPlan plan;
        plan.s2_levels.assign(s2_levels, s2_levels + n_levels);
        put_counters(predict_ddrgf_counters(l, plan), out);
    });
}
int ref_ddrgf_divides_evenly(long long l, const int* s2_levels, int n_levels) {
    DomainPlan plan;
    plan.s2_levels.assign(s2_levels, s2_levels + n_levels);
    return ddrgf_divides_evenly(l, plan) ? 1 : 0;
}

// interleave_permutation (partition.hpp:39-75): order[l], interior/separator
// groups as (first, count) pairs; returns the number of tasks or -1.
int ref_interleave_permutation(int l, int s1, int s2, int* order, int* interior, int* separator) {
    int n = -1;
    int rc = guarded(nullptr, [&] {
        auto lay = make_layout(l, 1, 1);
        auto [perm, desc] = interleave_permutation(lay, s1, s2);
        for (int p = 0; p < l; ++p) order[p] = perm.to_original[p];
        n = desc.n_tasks();
        for (int t = 0; t < n; ++t) {
            interior[2 * t] = desc.interior_groups[t].first;
            interior[2 * t + 1] = desc.interior_groups[t].count;
            separator[2 * t] = desc.separator_groups[t].first;
            separator[2 * t + 1] = desc.separator_groups[t].count;
        }
    });
    return rc == 0 ? n : -1;
}

// Cost model (cost_model.hpp:67-230) for pinning the product's restatement.
// kind 0 rgf(l), 1 nrgf(l, w), 2 fused(l, w), 3 ddrgf(l, plan); out = {gemm_eq, seconds}.
int ref_cost(int kind, long long l, long long w, const int* s2_levels, int n_levels, int n_threads,
             int terminal_threads, double r_lu, double r_getrs, double t_gemm, int blas_cap, double* out) {
    return guarded(nullptr, [&] {
        KernelRatios r{64, t_gemm, r_lu, r_getrs, 1};
        CostEstimate e;
        if (kind == 0) e = cost_rgf(l, r);
        else if (kind == 1) e = cost_nrgf(l, w, r);
        else if (kind == 2) e = cost_fused(l, w, r);
        else {
            DomainPlan plan;
            plan.s2_levels.assign(s2_levels, s2_levels + n_levels);
            plan.n_threads = n_threads;
            plan.terminal_threads = terminal_threads;
            e = cost_ddrgf(l, plan, r, blas_cap);
        }
        out[0] = e.gemm_equivalents;
        out[1] = e.predicted_seconds;
    });
}

// autotune (cost_model.hpp:174-224): ints = {use_rgf, ddrgf_valid, n_levels, terminal_threads,
// s2_0, s2_1, ...}; dbl = {rgf gemm_eq, ddrgf gemm_eq}.
int ref_autotune(long long l, int n_threads, double r_lu, double r_getrs, double t_gemm, int max_levels,
                 int s2_max, int blas_cap, int* ints, int max_ints, double* dbl) {
    return guarded(nullptr, [&] {
        KernelRatios r{64, t_gemm, r_lu, r_getrs, 1};
        TuneResult t = autotune(l, n_threads, r, max_levels, s2_max, blas_cap);
        ints[0] = t.use_rgf;
        ints[1] = t.ddrgf_valid;
        ints[2] = int(t.plan.s2_levels.size());
        ints[3] = t.plan.terminal_threads;
        for (size_t k = 0; k < t.plan.s2_levels.size() && int(4 + k) < max_ints; ++k) ints[4 + k] = t.plan.s2_levels[k];
        dbl[0] = t.rgf_cost.gemm_equivalents;
        dbl[1] = t.ddrgf_valid ? t.ddrgf_cost.gemm_equivalents : 0.0;
    });
}

}  // extern "C"
