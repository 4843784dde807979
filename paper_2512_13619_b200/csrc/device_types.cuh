// POD views handed to kernels by value, and the host-side owners behind the opaque C handles.
#pragma once
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "host/discretization.hpp"

namespace hdgb {

// Everything a kernel needs to know about the discretisation (device pointers).
struct DiscView {
    int D, M, ne, nf, n_lfe, n_orient, pe, pf, qe, qf;
    int npe;  // M*pe
    int mpf;  // M*pf
    int nfl;  // n_lfe*mpf   trace dofs per element
    int nfs;  // n_lfe*pf    scalar trace dofs per element
    int ne_owned, nf_owned;  // domain decomposition: owned elements / faces come first (== ne / nf on one GPU)
    const int* elem_faces;   // ne x n_lfe
    const int* elem_side;    // ne x n_lfe
    const int* face_elems;   // nf x 2
    const int* face_lidx;    // nf x 2
    const int* face_orient;  // nf x 2
    const int* bnd_tag;      // nf
    const double* phi;       // pe x qe
    const double* dphi[3];   // pe x qe
    const double* psi;       // pf x qf
    const double* tphi;      // [((lf*n_orient+o)*qf + gc)*pe + i]
    const double* es_vol;    // pe = 64 only (else null): ring-stage images of phi, dphi_r for the streamed E / D_d sweep,
                             // [stage of 8 points][table][point][68]; points past qe repeat the last one
    const double* es_face;   // pe = 64 only: tphi rows padded to 68 doubles, [((lf*n_orient+o)*qf + gc)*68 + i]
    const double* wq;        // qe
    const double* wf;        // qf
    const double* elem_detjac;
    const double* elem_invjac;
    const double* elem_coords;
    const double* face_detjac;
    const double* face_coords;
    const double* face_normal;
    const double* minv_b[3];  // pe x pe per element
    const double* minv_c[3];  // pe x nfs per element
};

struct ModelView {
    int kind;
    double p[16];
    const double* forcing_q;    // [(e*qe+g)*M + m] or nullptr
    const double* dirichlet_q;  // [(f*qf+g)*M + m] or nullptr
};

}  // namespace hdgb

struct hdgb_disc {
    hdgb_ctx* ctx = nullptr;
    hdgb_dims dims{};
    hdgb::HostMesh mesh;
    int ne_owned = -1, nf_owned = -1;     // domain decomposition: owned entities come first
    int ne_interior = 0, nf_interior = 0; // leading owned elements / faces that touch no halo face (overlap window)
    std::vector<int64_t> face_gid;        // local -> global face id (empty: identity)
    int64_t nf_global = -1;
    hdgb::MasterElement me;
    hdgb::HostGeom geom;
    // device tables
    hdgb::DevBuf<int> elem_faces, elem_side, face_elems, face_lidx, face_orient, bnd_tag;
    hdgb::DevBuf<double> phi, dphi[3], psi, tphi, wq, wf, es_vol, es_face;
    hdgb::DevBuf<double> elem_detjac, elem_invjac, elem_coords, face_detjac, face_coords, face_normal;
    hdgb::DevBuf<double> mass, mass_inv, bmat[3], cmat[3], minv_b[3], minv_c[3];
    hdgb::DiscView view{};
    double assemble_budget = 0.0;  // bytes of raw-block workspace per assembly chunk, fixed at the first assembly
    // residual-assembly workspace (assemble_residual runs once per line-search trial)
    hdgb::DevBuf<double> res_ruhat_e, res_partial, res_sums;
};

struct hdgb_model {
    hdgb_ctx* ctx = nullptr;
    hdgb::DevBuf<double> forcing_q, dirichlet_q;
    hdgb::ModelView view{};
    int n_comp = 1;
};

struct hdgb_state {
    hdgb_ctx* ctx = nullptr;
    const hdgb_disc* disc = nullptr;
    hdgb::DevBuf<double> u, uhat, q[3];
};

struct hdgb_ops {
    hdgb_ctx* ctx = nullptr;
    int npe = 0, nfl = 0, ne = 0, D = 0;
    hdgb::DevBuf<double> kbar, ebar_inv, fbar, hbar, rbar, ru, ruhat_e;
    bool has_raw = false;
    hdgb::DevBuf<double> e_raw, f_raw, h_raw, j_raw, d_raw[3], g_raw[3];
};

namespace hdgb {
// GMRES workspace, cached on the matrix (sized for one n_dof and restart length).
struct GmresWork {
    int restart = 0;
    int64_t n = 0;
    DevBuf<double> basis;    // (restart + 1) x n
    DevBuf<double> kv, r;    // n each
    DevBuf<double> coef;     // 2*(restart+1) + 2 device scalars: c | d | norm2
    DevBuf<double> partial;  // reduction workspace
    DevBuf<double> ycoef;    // restart device coefficients for the solution update
    DevBuf<double> cgs;      // workspace of the streamed CGS2 passes (ticket word + per-CTA partials)
};
}  // namespace hdgb

struct hdgb_matrix {
    hdgb_ctx* ctx = nullptr;
    std::unique_ptr<hdgb::GmresWork> work;
    bool neighbor_valid = false;
    int m = 1, pf = 0, n_lfe = 4, nf = 0;
    int nf_local = 0;  // faces a vector spans (owned first, then halo); == nf on one GPU
    int64_t spec_dummy = 0;  // stand-in operator counter of preconditioner-free solves (speculative GMRES pipelining)
    int nf_interior = 0;  // leading rows that reference owned faces only (computed while the halo exchange is in flight)
    int mpf() const { return m * pf; }
    int nb() const { return 2 * n_lfe - 1; }
    int64_t n_dof() const { return static_cast<int64_t>(mpf()) * nf; }          // owned unknowns (rows)
    int64_t n_local() const { return static_cast<int64_t>(mpf()) * nf_local; }  // vector length
    hdgb::DevBuf<double> blocks;           // mpf x (mpf*nb) per face
    hdgb::DevBuf<int> nbr32;               // nf x nb, device (kernels gather with 32-bit ids)
    std::vector<int64_t> neighbor;         // nf x nb, host, int64 with kNoFace = -1 (face_matrix.hpp:22)
    hdgb::DevBuf<double> rhs;              // optional
};

struct hdgb_precond {
    hdgb_ctx* ctx = nullptr;
    int kind = HDGB_PC_IDENTITY;
    int poly_degree = 0;
    int poly_kind = HDGB_POLY_GMRES;
    int mpf = 0, nf = 0, nf_local = 0, n_lfe = 0, ne = 0;
    hdgb::DevBuf<double> bj_inv;   // mpf^2 per face
    hdgb::DevBuf<double> asm_inv;  // nfl^2 per element
    const hdgb_disc* disc = nullptr;  // ASM gathers through the mesh tables
    std::vector<double> ritz;      // interleaved (re, im), Leja order
    int64_t inner_ops = 0;
    // work vectors
    hdgb::DevBuf<double> ze, wq, ww, wt, ws, wkv, yh;
};
