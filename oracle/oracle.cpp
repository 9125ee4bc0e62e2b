// ORACLE — plain, slow, obviously-correct CPU reference for the hot path of
// "Surface Multigrid via Intrinsic Prolongation" (arXiv 2104.13755).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.  It
// shares no code, header, table or helper with the CUDA product library
// (paper_2104_13755_b200/csrc); neither includes nor links the other.
//
// Single thread, IEEE binary64, built with -O2 -ffp-contract=off (reading
// A18 in DESIGN.md).  Citations: "P:n" = line n of /root/reference/PAPER.md.
// Readings of silent/garbled passages (A1..A22) are listed in DESIGN.md §3.
//
// Parity status per function (details in DESIGN.md §4 and tests/):
//   ora_cotan_laplacian   pinned (worked examples, FEM stiffness, L1=0, sphere closed form)
//   ora_lumped_mass       pinned (worked example, trace = area)
//   ora_prolongation      pinned (partition of unity, structure)
//   ora_galerkin          pinned (dense P^T A P via numpy, P=I, A=I, invariants)
//   ora_greedy_colouring  pinned (hand traces, brute-force properness)
//   ora_cholesky/_solve   pinned (worked examples, numpy.linalg)
//   ora_gs_sweep          pinned (worked example, A-norm decrease theorem)
//   ora_mg_vcycle         pinned (two-grid error-propagator formula, special cases)
//   ora_mg_solve          pinned (dense direct solve, closed forms)
//   ora_jacobi_sweep      pinned (worked example jacobi_2x2, splitting form vs numpy)
//   gs_sweep_reverse      pinned (the symmetric V-cycle operator is SPD; the forward one is not)
//   ora_mg_pcg            pinned (one level = one iteration, dense solve, CG energy monotonicity)
// oracle.py (numpy): dirichlet_reduce / dirichlet_solve pinned (no constraints =
// unconstrained, all known, dense constrained solve S:561, zero-column removal);
// bilaplacian pinned (Q1 = 0, symmetric PSD, 2-ring pattern, sphere Rayleigh
// quotient -> 4, dense smoothing solve).  Cycle / iteration COUNTS on the
// synthetic configs are parity unpinned (the paper prints none).

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <utility>
#include <vector>

namespace {

// ------------------------------------------------------------------------
// A compressed-sparse-row matrix, columns sorted ascending within each row.
struct Csr {
    int32_t nrows = 0, ncols = 0;
    std::vector<int64_t> rowptr;   // nrows + 1
    std::vector<int32_t> col;
    std::vector<double> val;
    int64_t nnz() const { return (int64_t)col.size(); }
};

// Build a sorted CSR from per-row (column, value) lists, summing duplicates in
// list order.
Csr from_rows(int32_t nrows, int32_t ncols, std::vector<std::vector<std::pair<int32_t, double>>>& rows) {
    Csr A;
    A.nrows = nrows;
    A.ncols = ncols;
    A.rowptr.assign(nrows + 1, 0);
    for (int32_t i = 0; i < nrows; ++i) {
        auto& r = rows[i];
        std::stable_sort(r.begin(), r.end(),
                         [](const std::pair<int32_t, double>& a, const std::pair<int32_t, double>& b) {
                             return a.first < b.first;
                         });
        for (size_t e = 0; e < r.size(); ++e) {
            if (e > 0 && r[e].first == r[e - 1].first) {
                A.val.back() += r[e].second;
            } else {
                A.col.push_back(r[e].first);
                A.val.push_back(r[e].second);
            }
        }
        A.rowptr[i + 1] = (int64_t)A.col.size();
    }
    return A;
}

// y = A x for one column (x, y strided by k).
double row_dot(const Csr& A, int32_t i, const double* x, int k, int c) {
    double s = 0.0;
    for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) s += A.val[e] * x[(int64_t)A.col[e] * k + c];
    return s;
}

double vec3_dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
void vec3_cross(const double* a, const double* b, double* o) {
    o[0] = a[1] * b[2] - a[2] * b[1];
    o[1] = a[2] * b[0] - a[0] * b[2];
    o[2] = a[0] * b[1] - a[1] * b[0];
}

// ------------------------------------------------------------------------
// Dense Cholesky, textbook row-by-row (Cholesky-Banachiewicz).  Alg. 2 "direct
// solve" at the coarsest level; reading A12: dense Cholesky, a
// non-positive pivot is an error.  L is n x n row-major, lower triangle used.
int dense_cholesky(int32_t n, const double* A, double* L) {
    for (int64_t t = 0; t < (int64_t)n * n; ++t) L[t] = 0.0;
    for (int32_t i = 0; i < n; ++i) {
        for (int32_t j = 0; j <= i; ++j) {
            double s = A[(int64_t)i * n + j];
            for (int32_t q = 0; q < j; ++q) s -= L[(int64_t)i * n + q] * L[(int64_t)j * n + q];
            if (i == j) {
                if (!(s > 0.0)) return 4;  // MG_ERR_NOT_SPD
                L[(int64_t)i * n + i] = std::sqrt(s);
            } else {
                L[(int64_t)i * n + j] = s / L[(int64_t)j * n + j];
            }
        }
    }
    return 0;
}

// Solve L L^T x = b (forward then backward substitution), k columns strided.
void dense_cholesky_solve(int32_t n, const double* L, int k, const double* B, double* X) {
    std::vector<double> y(n);
    for (int c = 0; c < k; ++c) {
        for (int32_t i = 0; i < n; ++i) {
            double s = B[(int64_t)i * k + c];
            for (int32_t q = 0; q < i; ++q) s -= L[(int64_t)i * n + q] * y[q];
            y[i] = s / L[(int64_t)i * n + i];
        }
        for (int32_t i = n - 1; i >= 0; --i) {
            double s = y[i];
            for (int32_t q = i + 1; q < n; ++q) s -= L[(int64_t)q * n + i] * X[(int64_t)q * k + c];
            X[(int64_t)i * k + c] = s / L[(int64_t)i * n + i];
        }
    }
}

// ------------------------------------------------------------------------
// Greedy graph colouring, Alg. 3 with App. A text.
// Readings: A6 descending degree, ties by ascending node index; A7 degree =
// number of distinct structural off-diagonal neighbours, palette scanned from
// the front, the chosen colour moved to the back, new colours appended, ids in
// creation order; A8 the structural pattern (stored zeros are edges).
int32_t greedy_colouring(const Csr& A, int32_t* colour) {
    const int32_t n = A.nrows;
    std::vector<int32_t> degree(n, 0);
    for (int32_t i = 0; i < n; ++i)
        for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e)
            if (A.col[e] != i) degree[i] += 1;   // columns are unique per row
    // "sort nodes {n_i} by degree", "descending order of degree"
    std::vector<int32_t> order(n);
    for (int32_t i = 0; i < n; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(),
                     [&](int32_t a, int32_t b) { return degree[a] > degree[b]; });
    for (int32_t i = 0; i < n; ++i) colour[i] = -1;
    std::vector<int32_t> palette;          // "pallette <- {}"
    int32_t ncolours = 0;
    std::vector<char> in_N;
    for (int32_t idx = 0; idx < n; ++idx) {
        const int32_t v = order[idx];
        // "N <- gather colors from painted neighbors of n_i"
        in_N.assign(ncolours, 0);
        for (int64_t e = A.rowptr[v]; e < A.rowptr[v + 1]; ++e) {
            int32_t u = A.col[e];
            if (u != v && colour[u] >= 0) in_N[colour[u]] = 1;
        }
        // "c <- find first entry in pallette not occurring in N"
        int pos = -1;
        for (size_t p = 0; p < palette.size(); ++p)
            if (!in_N[palette[p]]) { pos = (int)p; break; }
        int32_t c;
        if (pos < 0) {
            // "c <- new color; append c to pallette"
            c = ncolours++;
            palette.push_back(c);
        } else {
            // "move c to back of pallette"
            c = palette[pos];
            palette.erase(palette.begin() + pos);
            palette.push_back(c);
        }
        colour[v] = c;                      // "paint n_i with color c"
    }
    return ncolours;
}

// ------------------------------------------------------------------------
// Galerkin coarse-grid approximation A_c = R A P with R = P^T (Eq. gca,
// P:277-279; stored hierarchy A_{h+1} = P^T A_h P).  Entry by entry
// from the definition A_c[I,J] = sum_i sum_j P[i,I] A[i,j] P[j,J]: for each
// coarse row I, each fine i with P[i,I] != 0, each stored (i,j) of A, each
// stored (j,J) of P.  The pattern is structural (reading A9): every (I,J)
// reached this way is stored, whatever its value.
Csr galerkin(const Csr& P, const Csr& A) {
    const int32_t nf = P.nrows, nc = P.ncols;
    // columns of P: for each coarse I the fine rows i with P[i,I] != 0 (ascending i)
    std::vector<std::vector<std::pair<int32_t, double>>> Pcol(nc);
    for (int32_t i = 0; i < nf; ++i)
        for (int64_t e = P.rowptr[i]; e < P.rowptr[i + 1]; ++e) Pcol[P.col[e]].push_back({i, P.val[e]});
    Csr C;
    C.nrows = nc;
    C.ncols = nc;
    C.rowptr.assign(nc + 1, 0);
    std::vector<double> acc(nc, 0.0);
    std::vector<char> hit(nc, 0);
    std::vector<int32_t> touched;
    for (int32_t I = 0; I < nc; ++I) {
        touched.clear();
        for (auto& pi : Pcol[I]) {
            const int32_t i = pi.first;
            const double PiI = pi.second;
            for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) {
                const int32_t j = A.col[e];
                const double Aij = A.val[e];
                for (int64_t f = P.rowptr[j]; f < P.rowptr[j + 1]; ++f) {
                    const int32_t J = P.col[f];
                    if (!hit[J]) { hit[J] = 1; acc[J] = 0.0; touched.push_back(J); }
                    acc[J] += PiI * Aij * P.val[f];
                }
            }
        }
        std::sort(touched.begin(), touched.end());
        for (int32_t J : touched) {
            C.col.push_back(J);
            C.val.push_back(acc[J]);
            hit[J] = 0;
        }
        C.rowptr[I + 1] = (int64_t)C.col.size();
    }
    return C;
}

// ------------------------------------------------------------------------
// Multicolour Gauss-Seidel sweep (App. A; reading A2): colours in
// ascending id, rows of one colour in ascending index,
//   x_i <- (b_i - sum_{j != i} a_ij x_j) / a_ii,   for every column.
void gs_sweep(const Csr& A, const std::vector<std::vector<int32_t>>& classes, int k, const double* B, double* X) {
    for (const auto& cls : classes) {
        for (int32_t i : cls) {
            for (int c = 0; c < k; ++c) {
                double s = B[(int64_t)i * k + c];
                double aii = 0.0;
                for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) {
                    const int32_t j = A.col[e];
                    if (j == i) aii = A.val[e];
                    else s -= A.val[e] * X[(int64_t)j * k + c];
                }
                X[(int64_t)i * k + c] = s / aii;
            }
        }
    }
}

// Reverse-order multicolour GS sweep: colours in DESCENDING id (rows of a
// colour ascending).  The post-relaxation of the symmetric V-cycle used as a
// CG preconditioner (future work P:738): with the reversed
// order the post-smoother is the adjoint of the pre-smoother, so the V-cycle
// is a symmetric operator.
void gs_sweep_reverse(const Csr& A, const std::vector<std::vector<int32_t>>& classes, int k, const double* B,
                      double* X) {
    for (size_t cc = classes.size(); cc-- > 0;) {
        for (int32_t i : classes[cc]) {
            for (int c = 0; c < k; ++c) {
                double s = B[(int64_t)i * k + c];
                double aii = 0.0;
                for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) {
                    const int32_t j = A.col[e];
                    if (j == i) aii = A.val[e];
                    else s -= A.val[e] * X[(int64_t)j * k + c];
                }
                X[(int64_t)i * k + c] = s / aii;
            }
        }
    }
}

// Damped Jacobi sweep (App. E, "(damped) Jacobi"; damping omega,
// SPEC reading 0.8): x_i <- x_i + omega (b_i - sum_j a_ij x_j) / a_ii, every
// row from the OLD iterate.
void jacobi_sweep(const Csr& A, int k, const double* B, double* X, double omega) {
    const int32_t n = A.nrows;
    std::vector<double> old(X, X + (size_t)n * k);
    for (int32_t i = 0; i < n; ++i)
        for (int c = 0; c < k; ++c) {
            double s = B[(int64_t)i * k + c];
            double aii = 0.0;
            for (int64_t e = A.rowptr[i]; e < A.rowptr[i + 1]; ++e) {
                if (A.col[e] == i) aii = A.val[e];
                s -= A.val[e] * old[(int64_t)A.col[e] * k + c];
            }
            X[(int64_t)i * k + c] = old[(int64_t)i * k + c] + omega * s / aii;
        }
}

// ------------------------------------------------------------------------
struct Level {
    Csr A;                                        // A_l
    Csr P;                                        // P_l : level l+1 -> level l (absent at H)
    std::vector<int32_t> colour;
    int32_t ncolours = 0;
    std::vector<std::vector<int32_t>> classes;    // rows grouped by colour, ascending
};

struct MG {
    std::vector<Level> lv;
    int mu_pre = 2, mu_post = 2;                  // V(2,2): P:504
    int smoother = 0;                             // 0 multicolour GS (reading A2), 1 damped Jacobi (App. E)
    double omega = 0.8;                           // Jacobi damping
    int symmetric = 0;                            // 1: post-relaxation in reverse colour order
    std::vector<double> Lfac;                     // dense Cholesky factor of A_H
    int status = 0;
    // wall-clock phase times in seconds (timing only, for bench.py's CPU
    // baseline: SURVEY §8(d.6)); [0] Galerkin (symbolic + numeric, all
    // levels), [1] colouring + classes, [2] coarsest Cholesky, [3] V-cycles
    // and [4] residual norms of the last ora_mg_solve
    double phase_s[5] = {0, 0, 0, 0, 0};
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void build_classes(Level& L) {
    L.classes.assign(L.ncolours, {});
    for (int32_t i = 0; i < L.A.nrows; ++i) L.classes[L.colour[i]].push_back(i);
}

// Alg. 2 with reading A1: the correction is added to the
// pre-relaxed iterate x'_old.
void vcycle(MG& mg, int h, int k, const double* b, double* x) {
    Level& L = mg.lv[h];
    const int32_t n = L.A.nrows;
    const int H = (int)mg.lv.size() - 1;
    if (h == H) {
        // "solve A x_new = b  // direct solve"; x_old ignored
        dense_cholesky_solve(n, mg.Lfac.data(), k, b, x);
        return;
    }
    // pre-relaxation
    for (int s = 0; s < mg.mu_pre; ++s) {
        if (mg.smoother == 1) jacobi_sweep(L.A, k, b, x, mg.omega);
        else gs_sweep(L.A, L.classes, k, b, x);
    }
    // r_{h+1} <- P^T (b - A x'_old)
    std::vector<double> r((size_t)n * k);
    for (int32_t i = 0; i < n; ++i)
        for (int c = 0; c < k; ++c) r[(size_t)i * k + c] = b[(size_t)i * k + c] - row_dot(L.A, i, x, k, c);
    const int32_t nc = L.P.ncols;
    std::vector<double> rc((size_t)nc * k, 0.0);
    for (int32_t i = 0; i < n; ++i)
        for (int64_t e = L.P.rowptr[i]; e < L.P.rowptr[i + 1]; ++e)
            for (int c = 0; c < k; ++c) rc[(size_t)L.P.col[e] * k + c] += L.P.val[e] * r[(size_t)i * k + c];
    // c_{h+1} <- V-cycle(P^T A P, 0, r_{h+1}, h+1)
    std::vector<double> cc((size_t)nc * k, 0.0);
    vcycle(mg, h + 1, k, rc.data(), cc.data());
    // c_h <- P c_{h+1}; x'_new <- x'_old + c_h  (reading A1)
    for (int32_t i = 0; i < n; ++i)
        for (int c = 0; c < k; ++c) {
            double s = 0.0;
            for (int64_t e = L.P.rowptr[i]; e < L.P.rowptr[i + 1]; ++e) s += L.P.val[e] * cc[(size_t)L.P.col[e] * k + c];
            x[(size_t)i * k + c] += s;
        }
    // post-relaxation
    for (int s = 0; s < mg.mu_post; ++s) {
        if (mg.smoother == 1) jacobi_sweep(L.A, k, b, x, mg.omega);
        else if (mg.symmetric) gs_sweep_reverse(L.A, L.classes, k, b, x);
        else gs_sweep(L.A, L.classes, k, b, x);
    }
}

// rho_j = ||b_j - A x_j||_2 / ||b_j||_2 (reading A3; absolute norm if ||b_j|| = 0)
void residual_norms(const Csr& A, int k, const double* B, const double* X, const std::vector<double>& bnorm, double* out) {
    std::vector<double> ss(k, 0.0);
    for (int32_t i = 0; i < A.nrows; ++i)
        for (int c = 0; c < k; ++c) {
            double r = B[(size_t)i * k + c] - row_dot(A, i, X, k, c);
            ss[c] += r * r;
        }
    for (int c = 0; c < k; ++c) out[c] = std::sqrt(ss[c]) / (bnorm[c] > 0.0 ? bnorm[c] : 1.0);
}

}  // namespace

// ==========================================================================
// C ABI for the Python test harness (oracle/oracle.py).
extern "C" {

typedef struct Csr ora_csr;
typedef struct MG ora_mg;

ora_csr* ora_csr_new(int32_t nrows, int32_t ncols, const int64_t* rowptr, const int32_t* col, const double* val) {
    Csr* A = new Csr;
    A->nrows = nrows;
    A->ncols = ncols;
    A->rowptr.assign(rowptr, rowptr + nrows + 1);
    A->col.assign(col, col + rowptr[nrows]);
    A->val.assign(val, val + rowptr[nrows]);
    return A;
}
void ora_csr_free(ora_csr* A) { delete A; }
int32_t ora_csr_rows(const ora_csr* A) { return A->nrows; }
int32_t ora_csr_cols(const ora_csr* A) { return A->ncols; }
int64_t ora_csr_nnz(const ora_csr* A) { return A->nnz(); }
void ora_csr_export(const ora_csr* A, int64_t* rowptr, int32_t* col, double* val) {
    std::memcpy(rowptr, A->rowptr.data(), sizeof(int64_t) * (A->nrows + 1));
    std::memcpy(col, A->col.data(), sizeof(int32_t) * A->nnz());
    std::memcpy(val, A->val.data(), sizeof(double) * A->nnz());
}

// Cotangent Laplacian, PSD convention (reading A13):
//   L_ij = -1/2 sum_{o opposite (i,j)} cot angle_o,  L_ii = -sum_{j != i} L_ij.
// Faces in index order; at corner o of edge (i,j),
//   cot = (v_i-v_o).(v_j-v_o) / |(v_i-v_o) x (v_j-v_o)|.
// Boundary edges get a single term: natural BC.
ora_csr* ora_cotan_laplacian(int32_t n, int32_t nf, const double* V, const int32_t* F) {
    std::vector<std::vector<std::pair<int32_t, double>>> rows(n);
    for (int32_t f = 0; f < nf; ++f) {
        for (int corner = 0; corner < 3; ++corner) {
            const int32_t o = F[3 * f + corner];
            const int32_t i = F[3 * f + (corner + 1) % 3];
            const int32_t j = F[3 * f + (corner + 2) % 3];
            double ei[3], ej[3], cr[3];
            for (int d = 0; d < 3; ++d) {
                ei[d] = V[3 * i + d] - V[3 * o + d];
                ej[d] = V[3 * j + d] - V[3 * o + d];
            }
            vec3_cross(ei, ej, cr);
            const double cot = vec3_dot(ei, ej) / std::sqrt(vec3_dot(cr, cr));
            rows[i].push_back({j, -0.5 * cot});
            rows[j].push_back({i, -0.5 * cot});
            rows[i].push_back({i, 0.5 * cot});
            rows[j].push_back({j, 0.5 * cot});
        }
    }
    return new Csr(from_rows(n, n, rows));
}

// Lumped (barycentric) mass, M_ii = 1/3 sum_{f ni i} area_f (reading A14).
void ora_lumped_mass(int32_t n, int32_t nf, const double* V, const int32_t* F, double* M) {
    for (int32_t i = 0; i < n; ++i) M[i] = 0.0;
    for (int32_t f = 0; f < nf; ++f) {
        const int32_t a = F[3 * f], b = F[3 * f + 1], c = F[3 * f + 2];
        double e1[3], e2[3], cr[3];
        for (int d = 0; d < 3; ++d) {
            e1[d] = V[3 * b + d] - V[3 * a + d];
            e2[d] = V[3 * c + d] - V[3 * a + d];
        }
        vec3_cross(e1, e2, cr);
        const double area = 0.5 * std::sqrt(vec3_dot(cr, cr));
        M[a] += area / 3.0;
        M[b] += area / 3.0;
        M[c] += area / 3.0;
    }
}

// A = mass_coeff * diag(M) + lap_coeff * L on L's pattern (L must store its diagonal).
ora_csr* ora_mass_plus_laplacian(const ora_csr* L, const double* M, double mass_coeff, double lap_coeff) {
    Csr* A = new Csr(*L);
    for (int32_t i = 0; i < A->nrows; ++i)
        for (int64_t e = A->rowptr[i]; e < A->rowptr[i + 1]; ++e) {
            A->val[e] = lap_coeff * L->val[e];
            if (A->col[e] == i) A->val[e] += mass_coeff * M[i];
        }
    return A;
}

// y = A x, k columns (row-major n x k).
void ora_spmv(const ora_csr* A, int32_t k, const double* X, double* Y) {
    for (int32_t i = 0; i < A->nrows; ++i)
        for (int c = 0; c < k; ++c) Y[(size_t)i * k + c] = row_dot(*A, i, X, k, c);
}

// Linear barycentric prolongation P (n_fine x n_coarse), row i = the 3
// barycentric coordinates of fine vertex i in its coarse triangle.
// Entries with w == 0.0 are not stored (reading A9).
ora_csr* ora_prolongation(int32_t n_fine, int32_t n_coarse, const int32_t* cols, const double* w) {
    std::vector<std::vector<std::pair<int32_t, double>>> rows(n_fine);
    for (int32_t i = 0; i < n_fine; ++i)
        for (int q = 0; q < 3; ++q)
            if (w[3 * i + q] != 0.0) rows[i].push_back({cols[3 * i + q], w[3 * i + q]});
    return new Csr(from_rows(n_fine, n_coarse, rows));
}

ora_csr* ora_galerkin(const ora_csr* P, const ora_csr* A) { return new Csr(galerkin(*P, *A)); }

int32_t ora_greedy_colouring(const ora_csr* A, int32_t* colour) { return greedy_colouring(*A, colour); }

int ora_cholesky(int32_t n, const double* A, double* L) { return dense_cholesky(n, A, L); }
void ora_cholesky_solve(int32_t n, const double* L, int32_t k, const double* B, double* X) {
    dense_cholesky_solve(n, L, k, B, X);
}

void ora_gs_sweep(const ora_csr* A, const int32_t* colour, int32_t ncolours, int32_t k, const double* B, double* X) {
    std::vector<std::vector<int32_t>> classes(ncolours);
    for (int32_t i = 0; i < A->nrows; ++i) classes[colour[i]].push_back(i);
    gs_sweep(*A, classes, k, B, X);
}

// Setup (Alg. 1 lines 2-3 + stored hierarchy): P_l from ELL-3 arrays,
// A_{l+1} = P_l^T A_l P_l, Alg. 3 colouring of every level, dense Cholesky of
// A_H.  P_cols[l], P_w[l] are n_verts[l] x 3 and map level l+1 -> level l.
ora_mg* ora_mg_new(int32_t n_levels, const int32_t* n_verts, const int32_t* const* P_cols,
                   const double* const* P_w, const ora_csr* A0, int32_t mu_pre, int32_t mu_post) {
    MG* mg = new MG;
    mg->mu_pre = mu_pre;
    mg->mu_post = mu_post;
    mg->lv.resize(n_levels);
    mg->lv[0].A = *A0;
    double t0 = now_s();
    for (int l = 0; l + 1 < n_levels; ++l) {
        Csr* P = ora_prolongation(n_verts[l], n_verts[l + 1], P_cols[l], P_w[l]);
        mg->lv[l].P = *P;
        delete P;
        mg->lv[l + 1].A = galerkin(mg->lv[l].P, mg->lv[l].A);
    }
    double t1 = now_s();
    mg->phase_s[0] = t1 - t0;
    for (auto& L : mg->lv) {
        L.colour.resize(L.A.nrows);
        L.ncolours = greedy_colouring(L.A, L.colour.data());
        build_classes(L);
    }
    t0 = now_s();
    mg->phase_s[1] = t0 - t1;
    const Csr& AH = mg->lv.back().A;
    const int32_t nH = AH.nrows;
    std::vector<double> D((size_t)nH * nH, 0.0);
    for (int32_t i = 0; i < nH; ++i)
        for (int64_t e = AH.rowptr[i]; e < AH.rowptr[i + 1]; ++e) D[(size_t)i * nH + AH.col[e]] = AH.val[e];
    mg->Lfac.assign((size_t)nH * nH, 0.0);
    mg->status = dense_cholesky(nH, D.data(), mg->Lfac.data());
    mg->phase_s[2] = now_s() - t0;
    return mg;
}
void ora_mg_phase_times(const ora_mg* mg, double* out) { std::memcpy(out, mg->phase_s, sizeof(mg->phase_s)); }
void ora_mg_free(ora_mg* mg) { delete mg; }
int ora_mg_status(const ora_mg* mg) { return mg->status; }
int32_t ora_mg_levels(const ora_mg* mg) { return (int32_t)mg->lv.size(); }
void ora_mg_level_info(const ora_mg* mg, int32_t l, int32_t* n, int64_t* nnz, int32_t* ncolours) {
    *n = mg->lv[l].A.nrows;
    *nnz = mg->lv[l].A.nnz();
    *ncolours = mg->lv[l].ncolours;
}
void ora_mg_level_export(const ora_mg* mg, int32_t l, int64_t* rowptr, int32_t* col, double* val, int32_t* colour) {
    ora_csr_export(&mg->lv[l].A, rowptr, col, val);
    std::memcpy(colour, mg->lv[l].colour.data(), sizeof(int32_t) * mg->lv[l].A.nrows);
}
void ora_mg_coarse_factor(const ora_mg* mg, double* L) {
    std::memcpy(L, mg->Lfac.data(), sizeof(double) * mg->Lfac.size());
}

// One V-cycle at level 0 (Alg. 2), x updated in place.
void ora_mg_vcycle(ora_mg* mg, int32_t k, const double* B, double* X) { vcycle(*mg, 0, k, B, X); }

// Alg. 1 loop: rho_0, then V-cycles until every column has
// rho <= rel_tol (readings A3, A11) or max_cycles; rel_tol <= 0 runs exactly
// max_cycles.  hist[(c * k) + j] = rho of column j after cycle c.
// Returns 0 converged, 8 not converged, 7 NaN/Inf, 4 coarsest not SPD.
int ora_mg_solve(ora_mg* mg, int32_t k, const double* B, double* X, double rel_tol, int32_t max_cycles,
                 double* hist, int32_t* cycles_out) {
    if (mg->status != 0) return mg->status;
    const Csr& A = mg->lv[0].A;
    std::vector<double> bnorm(k, 0.0);
    for (int32_t i = 0; i < A.nrows; ++i)
        for (int c = 0; c < k; ++c) bnorm[c] += B[(size_t)i * k + c] * B[(size_t)i * k + c];
    for (int c = 0; c < k; ++c) bnorm[c] = std::sqrt(bnorm[c]);
    double tn = now_s();
    residual_norms(A, k, B, X, bnorm, hist);
    mg->phase_s[3] = 0.0;
    mg->phase_s[4] = now_s() - tn;
    int32_t cyc = 0;
    auto done = [&](const double* rho) {
        if (!(rel_tol > 0.0)) return false;
        for (int c = 0; c < k; ++c)
            if (!(rho[c] <= rel_tol)) return false;
        return true;
    };
    auto bad = [&](const double* rho) {
        for (int c = 0; c < k; ++c)
            if (!std::isfinite(rho[c])) return true;
        return false;
    };
    int rc = 8;
    if (bad(hist)) rc = 7;
    else if (done(hist)) rc = 0;
    while (rc == 8 && cyc < max_cycles) {
        const double tv = now_s();
        vcycle(*mg, 0, k, B, X);
        ++cyc;
        const double tr = now_s();
        residual_norms(A, k, B, X, bnorm, hist + (size_t)cyc * k);
        mg->phase_s[3] += tr - tv;
        mg->phase_s[4] += now_s() - tr;
        if (bad(hist + (size_t)cyc * k)) rc = 7;
        else if (done(hist + (size_t)cyc * k)) rc = 0;
    }
    *cycles_out = cyc;
    if (rc == 8 && !(rel_tol > 0.0)) rc = 0;   // fixed-cycle mode (config 1)
    return rc;
}

// Smoother selection: kind 0 multicolour GS, 1 damped Jacobi (omega);
// symmetric = 1 runs the post-relaxation colours in reverse order.
void ora_mg_set_smoother(ora_mg* mg, int32_t kind, double omega, int32_t symmetric) {
    mg->smoother = kind;
    mg->omega = omega;
    mg->symmetric = symmetric;
}

void ora_jacobi_sweep(const ora_csr* A, int32_t k, const double* B, double* X, double omega) {
    jacobi_sweep(*A, k, B, X, omega);
}

// Multigrid-preconditioned conjugate gradients ("use our
// multigrid solver as the pre-conditioner for ... the conjugate gradient
// method").  Textbook PCG, every column independently:
//   r = b - A x, z = M^{-1} r, p = z;  repeat: q = A p, alpha = (r,z)/(p,q),
//   x += alpha p, r -= alpha q, z = M^{-1} r, beta = (r,z)_new/(r,z)_old,
//   p = z + beta p.
// M^{-1} r = one V-cycle from a zero guess with the symmetric smoother
// ordering (forced here).  hist[(it * k) + j] = ||r_it||_2 / ||b_j||_2 of the
// recursively updated residual; stops when every column <= rel_tol.
// Returns 0 converged, 8 not converged, 7 NaN/Inf, 4 coarsest not SPD.
int ora_mg_pcg(ora_mg* mg, int32_t k, const double* B, double* X, double rel_tol, int32_t max_iters, double* hist,
               int32_t* iters_out) {
    if (mg->status != 0) return mg->status;
    const int sym_saved = mg->symmetric;
    mg->symmetric = 1;
    const Csr& A = mg->lv[0].A;
    const int32_t n = A.nrows;
    const size_t nk = (size_t)n * k;
    std::vector<double> r(nk), z(nk), p(nk), q(nk);
    std::vector<double> bnorm(k, 0.0), rz(k), pq(k), rr(k);
    for (size_t t = 0; t < nk; ++t) bnorm[t % k] += B[t] * B[t];
    for (int c = 0; c < k; ++c) bnorm[c] = std::sqrt(bnorm[c]);
    for (int32_t i = 0; i < n; ++i)
        for (int c = 0; c < k; ++c) r[(size_t)i * k + c] = B[(size_t)i * k + c] - row_dot(A, i, X, k, c);
    auto record = [&](int it) {
        std::fill(rr.begin(), rr.end(), 0.0);
        for (size_t t = 0; t < nk; ++t) rr[t % k] += r[t] * r[t];
        bool fin = true, done = rel_tol > 0.0;
        for (int c = 0; c < k; ++c) {
            const double v = std::sqrt(rr[c]) / (bnorm[c] > 0.0 ? bnorm[c] : 1.0);
            hist[(size_t)it * k + c] = v;
            fin &= std::isfinite(v);
            done &= v <= rel_tol;
        }
        return !fin ? 7 : done ? 0 : 8;
    };
    int rc = record(0);
    int32_t it = 0;
    while (rc == 8 && it < max_iters) {
        std::fill(z.begin(), z.end(), 0.0);
        vcycle(*mg, 0, k, r.data(), z.data());
        std::vector<double> rz_new(k, 0.0);
        for (size_t t = 0; t < nk; ++t) rz_new[t % k] += r[t] * z[t];
        for (size_t t = 0; t < nk; ++t) {
            const int c = (int)(t % k);
            const double beta = (it == 0 || rz[c] == 0.0) ? 0.0 : rz_new[c] / rz[c];   // reading A27
            p[t] = z[t] + beta * p[t];
        }
        rz = rz_new;
        std::fill(pq.begin(), pq.end(), 0.0);
        for (int32_t i = 0; i < n; ++i)
            for (int c = 0; c < k; ++c) {
                q[(size_t)i * k + c] = row_dot(A, i, p.data(), k, c);
                pq[c] += p[(size_t)i * k + c] * q[(size_t)i * k + c];
            }
        for (size_t t = 0; t < nk; ++t) {
            const int c = (int)(t % k);
            const double alpha = pq[c] == 0.0 ? 0.0 : rz[c] / pq[c];   // reading A27: solved column
            X[t] += alpha * p[t];
            r[t] -= alpha * q[t];
        }
        ++it;
        rc = record(it);
    }
    mg->symmetric = sym_saved;
    *iters_out = it;
    if (rc == 8 && !(rel_tol > 0.0)) rc = 0;
    return rc;
}

}  // extern "C"
