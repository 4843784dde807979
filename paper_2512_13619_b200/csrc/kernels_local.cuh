// Launchers of the element-local and global-assembly kernels.
#pragma once
#include "device_types.cuh"
#include "kernels.cuh"

namespace hdgb {

struct LocalIn {
    const double* u;
    const double* q[3];
    const double* uhat;
    const double* u_prev;  // nullptr when steady
    double dt_inv;         // 0 when steady
};

struct LocalOut {
    double* ru;
    double* ruhat_e;
    double* E;
    double* F;
    double* H;
    double* J;
    double* Dm[3];
    double* G[3];
};

// mass, B_d, C_d (local_ops.cpp:252-337)
void launch_local_factors(hdgb_ctx* ctx, const DiscView& dv, double* mass, double* const bmat[3], double* const cmat[3]);
// assemble_core (local_ops.cpp:33-228)
void launch_local_assemble(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in,
                           const LocalOut& out, bool want_jac);

// assemble_global (face_matrix.cpp:11-61): blocks (mpf x mpf*nb per face), rhs (mpf per face),
// neighbour table (int32 on device; the int64 host copy is derived from the mesh).
void launch_assemble_global(hdgb_ctx* ctx, const DiscView& dv, const double* kbar, const double* rbar,
                            double* blocks, double* rhs);
void launch_fill_neighbors(hdgb_ctx* ctx, const DiscView& dv, int* nbr32);
// build_bj extraction (preconditioner.cpp:33-37): diag[f] = slot-0 block of face f
void launch_extract_diag(hdgb_ctx* ctx, const double* blocks, int nf, int mpf, int nb, double* diag);
// build_asm enrichment (preconditioner.cpp:54-75): pbar = kbar with the diagonal sub-block of every
// local face replaced by that face's two-sided sum diag[f] (= the self block of the assembled row)
void launch_asm_enrich(hdgb_ctx* ctx, const DiscView& dv, const double* kbar, const double* diag, double* pbar);

}  // namespace hdgb
