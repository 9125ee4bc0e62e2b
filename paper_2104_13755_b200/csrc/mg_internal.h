// libmg internals shared by the host control plane (mg_host.cpp) and the
// sm_100a kernels (mg_kernels.cu).  Nothing here is visible through the C ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace mg {

constexpr int kMaxK = 4;          // right-hand sides per solve supported by the kernels
constexpr int kProfClasses = 11;  // see mg.h mg_get_profile
constexpr int kProfLevels = 16;

enum ProfClass {
    PC_GS = 0, PC_RESTRICT = 1, PC_PROLONG = 2, PC_COARSE = 3, PC_RESNORM = 4,
    PC_GALERKIN = 5, PC_ASSEMBLY = 6, PC_FACTOR = 7, PC_PERMUTE = 8, PC_TAIL = 9, PC_ALPHA = 10
};

// Device buffer owned by the context.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    cudaError_t alloc(size_t count) {
        if (count <= n && p) return cudaSuccess;
        release();
        if (count == 0) return cudaSuccess;
        cudaError_t e = cudaMalloc(&p, count * sizeof(T));
        if (e == cudaSuccess) n = count;
        return e;
    }
    cudaError_t upload(const std::vector<T>& v, cudaStream_t s) {
        cudaError_t e = alloc(v.size());
        if (e != cudaSuccess || v.empty()) return e;
        return cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    }
};

// One grid of the hierarchy.  "internal" order = rows grouped by Alg. 3
// colour (ascending), locality (Morton) order inside a colour; the coarsest
// level keeps the user order (it has no smoother).
struct Level {
    int32_t n = 0;
    int64_t nnz = 0;
    int32_t ncolours = 0;
    int lpr = 8;                          // lanes per row of the CSR kernels (untiled fallback)
    int lpr_all = 4;                      // lanes per row of whole-level passes (residual, norm)
    bool tiled = false;                   // tile-staged kernels usable (tiles fit in shared memory)
    int cap_gs = 0;                       // max nnz of a kTile-row tile inside one colour range
    int cap_all = 0;                      // max nnz of a kTile-row tile of the whole matrix
    bool pipe = false;                    // persistent TMA-bulk pipelined tile kernels
    int pipe_cap = 0;                     // max nnz of any tile (GS or whole-level tiles)
    mutable int pass_ctr = 0;             // pipelined launches enqueued on this level (serpentine direction)
    bool serpentine = true;               // alternate the tile walk direction between passes
    bool restrict_ordered = true;         // (this level coarse) restriction visits rows in gal_order
    DBuf<int32_t> rcptr, rcidx;           // children lists in gal_order (ordered restriction)
    DBuf<double> rcw;
    bool pipe_unr8 = false;               // k_tile_pipe with 8 gathers per batch (K = 3, 3 CTAs/SM)
    int pipe_lpr = 1;
                     // lanes per row of the pipelined tiles (tiles of kTile / pipe_lpr rows)
    std::vector<int32_t> tile_off;        // tiles of colour c: [tile_off[c], tile_off[c+1]); whole level: last range
                                          // (set balanced for 3 resident CTAs per SM)
    std::vector<int32_t> tile_off4;       // the same for 4 resident CTAs per SM (second set in `tiles`)
    DBuf<int32_t> tiles;                  // {row0, nrow, e0, e1} per tile
    std::vector<double> V;                // user-order positions [n][3]
    std::vector<int32_t> colour;          // user order
    std::vector<int32_t> colour_off;      // internal row ranges per colour [ncolours+1]
    std::vector<int32_t> perm, iperm;     // perm[internal] = user, iperm[user] = internal
    std::vector<int32_t> urp, ucol;       // user-order CSR pattern
    std::vector<int32_t> irp, icol;       // internal CSR pattern
    std::vector<int64_t> i2u;             // internal nnz -> user nnz
    // ELL-3 prolongation P_l (this level fine, next level coarse), user order
    std::vector<int32_t> Pc_user;
    std::vector<double> Pw_user;

    DBuf<int32_t> rp, col;                // internal CSR pattern
    DBuf<double> val;                     // internal values
    DBuf<double> qv, mv;                  // App. D split operators Q_l, M_l (internal order, same pattern)
    DBuf<int32_t> pc;                     // P_l SoA [3][n], coarse internal column
    DBuf<double> pw;                      // P_l SoA [3][n]
    DBuf<int32_t> cptr, cidx;             // transpose of P_{l-1} (this level coarse): children
    DBuf<double> cw;
    DBuf<int32_t> gal_order;              // rows of this level in locality order (Galerkin)
    // numeric Galerkin k_galerkin_t (this level coarse; structure built by
    // build_galerkin_t in mg_host.cpp, integer data only)
    int galt_tcap = 0;                    // 16 / 32: T-positions per fine row; 0: generic kernel
    int galt_ngroups = 0;
    DBuf<int32_t> gt_rows, gt_uoff;       // groups: gal_order offsets, offsets into the distinct children (U)
    DBuf<int32_t> gt_ent, gt_con;         // groups: coarse-entry offsets, contribution offsets
    DBuf<uint16_t> gt_eoff;               // per entry (+1 sentinel per group): contribution offset in the group
    DBuf<uint8_t> gt_rowidx, gt_slot;     // per entry: local row in the group, column slot in the row
    DBuf<uint16_t> gt_codes;              // contributions: child u | T-position k << 8 | parent slot q << 13
    DBuf<int32_t> gt_umeta;               // per U row: {first nonzero, fine row, length, T length}
    DBuf<int32_t> gt_crp;                 // per gal_order row: first slot of the coarse row
    DBuf<uint16_t> gt_tp;                 // (this level fine) per nonzero: T-positions of the 3 parents of col
    DBuf<uint8_t> gt_tlen;                // (this level fine) T-pattern length per row
    DBuf<double> prow_w;                  // P rows packed: {w0, w1, w2, 0} (this level fine)
    DBuf<int32_t> dperm;                  // perm on device
    DBuf<int32_t> diperm;                 // iperm on device (user -> internal)
    DBuf<int64_t> di2u;                   // level 0: internal nnz -> user nnz
    DBuf<double> x, b, r;                 // [n][kMaxK] work vectors
};


// Device-side state of the V-cycle loop (mg_solve with the conditional graph).
struct LoopState {
    double tol;
    int max_cycles;
    int cyc;       // cycles run
    int status;    // 0 running / budget spent, 1 converged, 2 non-finite
    int pad;
};
constexpr int kLoopHistCycles = 4096;   // device history capacity (cycles)

// Launch helpers.  All enqueue on `s` and return the number of kernel
// launches issued.  `pdl`: launch with programmatic stream serialisation
// (V-cycle graph).
// mg_vcycle.cu
int vc_gs(int K, const Level& L, int r0, int r1, bool pdl, cudaStream_t s);          // one colour class
int vc_residual(int K, const Level& L, bool pdl, cudaStream_t s);
int vc_loop_check(int K, const double* rho, LoopState* st, double* hist, cudaGraphConditionalHandle h, cudaStream_t s);
int vc_jacobi(int K, const Level& L, double* xin, double* xout, double omega, bool pdl, cudaStream_t s);  // xout = xin + omega D^-1 (b - A xin)                    // L.r = L.b - A L.x
int vc_restrict(int K, const Level& coarse, const Level& fine, bool pdl, cudaStream_t s);  // coarse.b = P^T fine.r, coarse.x = 0
int vc_prolong(int K, const Level& fine, const Level& coarse, bool pdl, cudaStream_t s);   // fine.x += P coarse.x
int vc_coarse_gemv(int K, const double* Z, int npad, int n, const double* b, double* x, bool pdl, cudaStream_t s);
int vc_coarse_trsv(int K, const double* L, const double* Linv, int npad, int n, const double* b, double* x, bool pdl,
                   cudaStream_t s);
int vc_resnorm(int K, const Level& L, double* partial, int nb, const double* bnorm, double* rho, bool pdl,
               cudaStream_t s);
int vc_sumsq(int K, const double* v, int n, double* partial, int nb, double* out, cudaStream_t s);
int vc_norm_finalize(int K, const double* partial, int nb, const double* denom, double* out, bool pdl, cudaStream_t s);
int resnorm_blocks(int n);
int tile_rows();
size_t tile_smem_limit();
size_t pipe_smem_bytes(int cap);
void init_vcycle_attributes();
// mg_krylov.cu (MG-preconditioned CG, row f4)
int pcg_blocks();
int pcg_update_blocks(int n);
int pcg_prep(int K, const double* r, double* b0, double* x0, int n, bool pdl, cudaStream_t s);
int pcg_direction(int K, const double* r, const double* z, double* p, int n, double* partial, double* sc, int* first,
                  bool pdl, cudaStream_t s);
int pcg_step(int K, const Level& L0, double* x, double* r, const double* p, double* q, double* partial, double* sc,
             bool pdl, cudaStream_t s);
// mg_setup.cu
void init_setup_attributes();
int launch_gather_rows(int K, const int32_t* iperm, const double* src_user, double* dst_int, int n, cudaStream_t s,
                       const int32_t* umap = nullptr);
int launch_scatter_rows(int K, const int32_t* iperm, const double* src_int, double* dst_user, int n, cudaStream_t s,
                        const int32_t* umap = nullptr);
int launch_dirichlet_rhs(int K, const int32_t* krp, const int32_t* kcol, const double* kval, const double* X,
                         double* b, int n, cudaStream_t s);
int launch_gather_vals(const int64_t* i2u, const double* src, double* dst, int64_t nnz, cudaStream_t s);
int launch_cotan(const Level& L0, const int32_t* opp, const uint8_t* opp8, const double* Vint, double mass_coeff, double lap_coeff,
                 double* val, double* M_int, cudaStream_t s);
int launch_bilaplacian(const int32_t* rp2, const int32_t* col2, const int32_t* rp1, const int32_t* col1,
                       const double* Lv, const double* M, double mass_coeff, double bilap_coeff, double* out, int n,
                       cudaStream_t s);
int launch_axpby(const double* Qv, const double* Mv, double alpha, double beta, double* out, int64_t nnz,
                 cudaStream_t s);
int launch_apply_mass(int K, const double* M_user, const double* X, double* B, int n, cudaStream_t s);
int launch_scatter_vec(const int32_t* iperm, const double* src_int, double* dst_user, int n, cudaStream_t s);
int launch_galerkin(const Level& fine, const double* fval, const Level& coarse, double* cval, cudaStream_t s);
int launch_densify(const Level& LH, double* D, int npad, cudaStream_t s);
int launch_chol_grid(double* D, double* Linv, double* W, double* Z, int npad, int* err, cudaStream_t s);

}  // namespace mg
