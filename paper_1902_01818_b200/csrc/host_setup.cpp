// host_setup.cpp -- native (OpenMP) host setup for the hierarchy build (libigb_setup.so).
//
// Setup stays on the host as in the reference (BASELINE north star); this file only makes the
// two setup steps that dominate the large configurations fast, with results BIT-IDENTICAL to the
// SciPy code paths they replace (tests/test_setup.py compares them array for array):
//
//  * igbs_kron_reduce: the Kronecker assembly of affine patches and its reduction to free DoFs,
//      reference assembly.py:333-344 (per patch K = sum_a c_a (x)_i (K_i if i == a else M_i))
//      followed by assembly.py:568-608 (COO of every patch mapped to free ids, tocsr);
//      replaces paper_1902_01818_b200.assembly._bulk_matrices (affine branch) + _coo_sum.
//      Arithmetic order reproduced: scipy kron data (x0 * x1) * x2, the scalar c_a applied
//      per term, the csr_plus_csr sums ((c0 t0 + c1 t1) + c2 t2) with exact zeros dropped,
//      coo_tocsr's row order (patches in order, each patch row in column order), then
//      csr_sort_indices (std::sort with a key-only comparator -- applied to every row iff some
//      row is not non-decreasing, as scipy's has_sorted_indices decides) and csr_sum_duplicates.
//  * igbs_galerkin: A_{l-1} = (P^T A) P, reference multigrid.py:95-99; replaces SciPy's two
//      csc_matmat calls (csr_matmat on the transposed operands): X[k,j] = sum_{m asc} A[m,j] P[m,k],
//      Y[k,i] = sum_{j asc} P[j,i] X[k,j], accumulated from 0.0 in that order, exact zeros dropped,
//      then returned as sorted CSR (Y.tocsr()).
//  * igbs_max_asym: the symmetry check of assembly.py:611-613 (max |A - A^T|, max |A|).
//
// Results live in an opaque handle: igbs_nnz() -> caller allocates -> igbs_copy() -> igbs_free().
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <utility>
#include <vector>

namespace {

struct Csr {
  int64_t n_rows = 0, n_cols = 0;
  std::vector<int64_t> ptr;  // final row pointers
  // entries of row r live at [src[r], src[r] + len) of col/val (raw, compacted by igbs_copy)
  std::vector<int64_t> src;
  std::vector<int32_t> col;
  std::vector<double> val;
};

// key-only comparator, as scipy's kv_pair_less (sparsetools/csr.h)
bool kv_pair_less(const std::pair<int32_t, double>& x, const std::pair<int32_t, double>& y) { return x.first < y.first; }

// Parallel deterministic transpose (CSR -> CSR of the transpose; entries of each output row in
// ascending source-row order, exactly what csr_tocsc produces).
void transpose(int64_t n_rows, int64_t n_cols, const int64_t* ptr, const int32_t* col, const double* val,
               std::vector<int64_t>& tptr, std::vector<int32_t>& tcol, std::vector<double>& tval) {
  const int T = omp_get_max_threads();
  std::vector<int64_t> bounds(T + 1);
  for (int t = 0; t <= T; ++t) bounds[t] = n_rows * t / T;
  std::vector<std::vector<int64_t>> cnt(T, std::vector<int64_t>(n_cols + 1, 0));
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    auto& c = cnt[t];
    for (int64_t r = bounds[t]; r < bounds[t + 1]; ++r)
      for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) ++c[col[k]];
  }
  tptr.assign(n_cols + 1, 0);
  // offsets: column j, thread t starts after columns < j and threads < t
  int64_t run = 0;
  for (int64_t j = 0; j < n_cols; ++j) {
    tptr[j] = run;
    for (int t = 0; t < T; ++t) {
      const int64_t c = cnt[t][j];
      cnt[t][j] = run;
      run += c;
    }
  }
  tptr[n_cols] = run;
  tcol.resize(run);
  tval.resize(run);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    auto& c = cnt[t];
    for (int64_t r = bounds[t]; r < bounds[t + 1]; ++r)
      for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
        const int64_t at = c[col[k]]++;
        tcol[at] = (int32_t)r;
        tval[at] = val[k];
      }
  }
}

}  // namespace

extern "C" {

int igbs_num_threads(void) { return omp_get_max_threads(); }

int64_t igbs_nnz(void* h) { return static_cast<Csr*>(h)->ptr.back(); }

// Copy the result into caller buffers: indptr (int32 if idx64 == 0 else int64), indices, data.
void igbs_copy(void* h, void* indptr, int idx64, int32_t* indices, double* data) {
  Csr& C = *static_cast<Csr*>(h);
  const int64_t n = C.n_rows;
  if (idx64) {
    std::memcpy(indptr, C.ptr.data(), sizeof(int64_t) * (n + 1));
  } else {
    int32_t* p = static_cast<int32_t*>(indptr);
    for (int64_t r = 0; r <= n; ++r) p[r] = (int32_t)C.ptr[r];
  }
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < n; ++r) {
    const int64_t len = C.ptr[r + 1] - C.ptr[r];
    std::memcpy(indices + C.ptr[r], C.col.data() + C.src[r], sizeof(int32_t) * len);
    std::memcpy(data + C.ptr[r], C.val.data() + C.src[r], sizeof(double) * len);
  }
}

void igbs_free(void* h) { delete static_cast<Csr*>(h); }

// Kronecker assembly of affine patches reduced to free DoFs (see the file header).
//   dim in {2,3}; npatch patches; block_off[npatch+1] block offsets; dims[npatch*dim];
//   c[npatch*dim] = det / s_a^2; per (patch, axis) q = k*dim + a the 1-D CSR pattern
//   ip[ptr_off[q] .. + dims+1], ix[ent_off[q] ..] shared by mass mval and stiffness kval;
//   row_map / col_map [n_block]: block index -> free (row) / column id or -1.
void* igbs_kron_reduce(int dim, int npatch, const int64_t* block_off, const int32_t* dims, const double* c,
                       const int64_t* ptr_off, const int64_t* ent_off, const int32_t* ip, const int32_t* ix,
                       const double* mval, const double* kval, const int32_t* row_map, const int32_t* col_map,
                       int64_t n_rows, int64_t n_cols) {
  const int64_t n_block = block_off[npatch];
  Csr* out = new Csr;
  Csr& C = *out;
  C.n_rows = n_rows;
  C.n_cols = n_cols;
  // copies of every free row in block order (= patch order, then local order): coo_tocsr order
  std::vector<int64_t> cp_ptr(n_rows + 1, 0);
  for (int64_t b = 0; b < n_block; ++b)
    if (row_map[b] >= 0) ++cp_ptr[row_map[b] + 1];
  for (int64_t r = 0; r < n_rows; ++r) cp_ptr[r + 1] += cp_ptr[r];
  std::vector<int64_t> cp(cp_ptr[n_rows]);
  {
    std::vector<int64_t> fill(cp_ptr.begin(), cp_ptr.end() - 1);
    for (int64_t b = 0; b < n_block; ++b)
      if (row_map[b] >= 0) cp[fill[row_map[b]]++] = b;
  }
  std::vector<int> patch_of_copy(cp.size());
  for (size_t i = 0; i < cp.size(); ++i)
    patch_of_copy[i] = (int)(std::upper_bound(block_off, block_off + npatch + 1, cp[i]) - block_off - 1);

  // enumerate the raw (pre-sum) entries of free row r in coo_tocsr order
  auto for_raw = [&](int64_t r, auto&& emit) {
    for (int64_t ci = cp_ptr[r]; ci < cp_ptr[r + 1]; ++ci) {
      const int k = patch_of_copy[ci];
      const int64_t loc = cp[ci] - block_off[k], off = block_off[k];
      const int32_t* dk = dims + (size_t)k * dim;
      const double* ck = c + (size_t)k * dim;
      int idx[3];
      int64_t rem = loc;
      for (int a = dim - 1; a >= 0; --a) {
        idx[a] = (int)(rem % dk[a]);
        rem /= dk[a];
      }
      const int q0 = k * dim;
      const int32_t* p0 = ip + ptr_off[q0];
      const int32_t* p1 = ip + ptr_off[q0 + 1];
      const int64_t e0 = ent_off[q0], e1 = ent_off[q0 + 1];
      if (dim == 2) {
        for (int32_t u = p0[idx[0]]; u < p0[idx[0] + 1]; ++u) {
          const int32_t j0 = ix[e0 + u];
          const double m0 = mval[e0 + u], k0 = kval[e0 + u];
          for (int32_t v = p1[idx[1]]; v < p1[idx[1] + 1]; ++v) {
            const int32_t j1 = ix[e1 + v];
            const double m1 = mval[e1 + v], k1 = kval[e1 + v];
            const int32_t cm = col_map[off + (int64_t)j0 * dk[1] + j1];
            if (cm < 0) continue;
            const double t0 = k0 * m1, t1 = m0 * k1;
            const double s = t0 * ck[0] + t1 * ck[1];
            if (s != 0.0) emit(cm, s);
          }
        }
      } else {
        const int32_t* p2 = ip + ptr_off[q0 + 2];
        const int64_t e2 = ent_off[q0 + 2];
        for (int32_t u = p0[idx[0]]; u < p0[idx[0] + 1]; ++u) {
          const int32_t j0 = ix[e0 + u];
          const double m0 = mval[e0 + u], k0 = kval[e0 + u];
          for (int32_t v = p1[idx[1]]; v < p1[idx[1] + 1]; ++v) {
            const int32_t j1 = ix[e1 + v];
            const double m1 = mval[e1 + v], k1 = kval[e1 + v];
            const double km = k0 * m1, mk = m0 * k1, mm = m0 * m1;
            const int64_t base = off + ((int64_t)j0 * dk[1] + j1) * dk[2];
            for (int32_t w = p2[idx[2]]; w < p2[idx[2] + 1]; ++w) {
              const int32_t j2 = ix[e2 + w];
              const int32_t cm = col_map[base + j2];
              if (cm < 0) continue;
              const double m2 = mval[e2 + w], k2 = kval[e2 + w];
              const double t0 = km * m2, t1 = mk * m2, t2 = mm * k2;
              const double s = (t0 * ck[0] + t1 * ck[1]) + t2 * ck[2];
              if (s != 0.0) emit(cm, s);
            }
          }
        }
      }
    }
  };

  // pass 1: raw counts and whether every raw row is non-decreasing (scipy has_sorted_indices)
  std::vector<int64_t> raw(n_rows + 1, 0);
  int unsorted = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : unsorted)
  for (int64_t r = 0; r < n_rows; ++r) {
    int64_t cnt = 0;
    int32_t last = -1;
    int bad = 0;
    for_raw(r, [&](int32_t cm, double) {
      bad |= cm < last;
      last = cm;
      ++cnt;
    });
    raw[r + 1] = cnt;
    unsorted |= bad;
  }
  for (int64_t r = 0; r < n_rows; ++r) raw[r + 1] += raw[r];
  C.src.assign(raw.begin(), raw.end() - 1);
  C.col.resize(raw[n_rows]);
  C.val.resize(raw[n_rows]);
  std::vector<int64_t> len(n_rows, 0);
  // pass 2: fill, sort (iff scipy would), sum duplicates left to right
#pragma omp parallel
  {
    std::vector<std::pair<int32_t, double>> tmp;
#pragma omp for schedule(dynamic, 256)
    for (int64_t r = 0; r < n_rows; ++r) {
      tmp.clear();
      for_raw(r, [&](int32_t cm, double s) { tmp.emplace_back(cm, s); });
      if (unsorted) std::sort(tmp.begin(), tmp.end(), kv_pair_less);
      int64_t o = raw[r], n = 0;
      for (size_t i = 0; i < tmp.size();) {
        const int32_t j = tmp[i].first;
        double x = tmp[i].second;
        ++i;
        while (i < tmp.size() && tmp[i].first == j) x += tmp[i++].second;
        C.col[o + n] = j;
        C.val[o + n] = x;
        ++n;
      }
      len[r] = n;
    }
  }
  C.ptr.assign(n_rows + 1, 0);
  for (int64_t r = 0; r < n_rows; ++r) C.ptr[r + 1] = C.ptr[r] + len[r];
  return out;
}

// Galerkin coarse operator (P^T A) P with SciPy's arithmetic (see the file header).
//   A: nf x nf CSR (int64 ptr, sorted indices); P: nf x nc CSR (sorted).
void* igbs_galerkin(int64_t nf, int64_t nc, const int64_t* a_ptr, const int32_t* a_col, const double* a_val,
                    const int64_t* p_ptr, const int32_t* p_col, const double* p_val) {
  // columns of A (entries in ascending row order) and of P
  std::vector<int64_t> at_ptr, pt_ptr;
  std::vector<int32_t> at_col, pt_col;
  std::vector<double> at_val, pt_val;
  transpose(nf, nf, a_ptr, a_col, a_val, at_ptr, at_col, at_val);
  transpose(nf, nc, p_ptr, p_col, p_val, pt_ptr, pt_col, pt_val);
  const int T = omp_get_max_threads();
  // X = P^T A, column j (fine) -> entries (k coarse, value), per-thread storage
  struct Span {
    int t;
    int64_t off, len;
  };
  std::vector<Span> xs(nf);
  std::vector<std::vector<int32_t>> xk(T);
  std::vector<std::vector<double>> xv(T);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    std::vector<double> acc(nc, 0.0);
    std::vector<char> seen(nc, 0);
    std::vector<int32_t> touched;
#pragma omp for schedule(dynamic, 512)
    for (int64_t j = 0; j < nf; ++j) {
      touched.clear();
      for (int64_t q = at_ptr[j]; q < at_ptr[j + 1]; ++q) {
        const int32_t m = at_col[q];
        const double v = at_val[q];  // A[m, j]
        for (int64_t e = p_ptr[m]; e < p_ptr[m + 1]; ++e) {
          const int32_t k = p_col[e];
          acc[k] += v * p_val[e];
          if (!seen[k]) {
            seen[k] = 1;
            touched.push_back(k);
          }
        }
      }
      std::sort(touched.begin(), touched.end());
      const int64_t off = (int64_t)xk[t].size();
      for (int32_t k : touched) {
        if (acc[k] != 0.0) {
          xk[t].push_back(k);
          xv[t].push_back(acc[k]);
        }
        acc[k] = 0.0;
        seen[k] = 0;
      }
      xs[j] = Span{t, off, (int64_t)xk[t].size() - off};
    }
  }
  // Y = X P, column i (coarse) -> entries (k, value)
  std::vector<Span> ys(nc);
  std::vector<std::vector<int32_t>> yk(T);
  std::vector<std::vector<double>> yv(T);
#pragma omp parallel num_threads(T)
  {
    const int t = omp_get_thread_num();
    std::vector<double> acc(nc, 0.0);
    std::vector<char> seen(nc, 0);
    std::vector<int32_t> touched;
#pragma omp for schedule(dynamic, 256)
    for (int64_t i = 0; i < nc; ++i) {
      touched.clear();
      for (int64_t q = pt_ptr[i]; q < pt_ptr[i + 1]; ++q) {
        const int32_t j = pt_col[q];
        const double v = pt_val[q];  // P[j, i]
        const Span& s = xs[j];
        const int32_t* kk = xk[s.t].data() + s.off;
        const double* vv = xv[s.t].data() + s.off;
        for (int64_t e = 0; e < s.len; ++e) {
          const int32_t k = kk[e];
          acc[k] += v * vv[e];
          if (!seen[k]) {
            seen[k] = 1;
            touched.push_back(k);
          }
        }
      }
      std::sort(touched.begin(), touched.end());
      const int64_t off = (int64_t)yk[t].size();
      for (int32_t k : touched) {
        if (acc[k] != 0.0) {
          yk[t].push_back(k);
          yv[t].push_back(acc[k]);
        }
        acc[k] = 0.0;
        seen[k] = 0;
      }
      ys[i] = Span{t, off, (int64_t)yk[t].size() - off};
    }
  }
  xk.clear();
  xv.clear();
  // Y as CSC (columns i) -> CSR rows k with ascending i (csc_tocsr order)
  std::vector<int64_t> y_ptr(nc + 1, 0);
  for (int64_t i = 0; i < nc; ++i) y_ptr[i + 1] = y_ptr[i] + ys[i].len;
  std::vector<int32_t> y_col(y_ptr[nc]);
  std::vector<double> y_val(y_ptr[nc]);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nc; ++i) {
    const Span& s = ys[i];
    std::memcpy(y_col.data() + y_ptr[i], yk[s.t].data() + s.off, sizeof(int32_t) * s.len);
    std::memcpy(y_val.data() + y_ptr[i], yv[s.t].data() + s.off, sizeof(double) * s.len);
  }
  yk.clear();
  yv.clear();
  Csr* out = new Csr;
  out->n_rows = nc;
  out->n_cols = nc;
  std::vector<int64_t> r_ptr;
  transpose(nc, nc, y_ptr.data(), y_col.data(), y_val.data(), r_ptr, out->col, out->val);
  out->ptr = r_ptr;
  out->src.assign(r_ptr.begin(), r_ptr.end() - 1);
  return out;
}

// max |A - A^T| over the union pattern and max |A| (assembly.py:611-613's symmetry check)
void igbs_max_asym(int64_t n, const int64_t* ptr, const int32_t* col, const double* val, double* max_asym,
                   double* max_abs) {
  double ma = 0.0, mb = 0.0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(max : ma, mb)
  for (int64_t r = 0; r < n; ++r) {
    for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) {
      const int32_t j = col[k];
      mb = std::max(mb, std::fabs(val[k]));
      const int32_t* b = col + ptr[j];
      const int32_t* e = col + ptr[j + 1];
      const int32_t* f = std::lower_bound(b, e, (int32_t)r);
      const double t = (f != e && *f == r) ? val[ptr[j] + (f - b)] : 0.0;
      ma = std::max(ma, std::fabs(val[k] - t));
    }
  }
  *max_asym = ma;
  *max_abs = mb;
}

}  // extern "C"
