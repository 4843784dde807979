// C ABI: the global face-block operator (A7-A8) and the preconditioners (A9-A12).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <random>

#include "host/ritz.hpp"
#include "solver.cuh"

using namespace hdgb;

namespace hdgb {

void matvec_device(hdgb_matrix* k, const double* x, double* y) {
    // block_matvec (face_matrix.cpp:83-107) with gather_extended (:63-81) fused into the GEMV:
    // the nb neighbour slices are staged in shared memory, the block row is streamed once.
    // Domain decomposition: the halo part of x is refreshed from its owners; the leading rows that reference owned
    // faces only (nf_interior) are computed while that exchange is in flight, the interface rows after it has landed.
    hdgb_ctx* c = k->ctx;
    const int mpf = k->mpf(), nb = k->nb();
    auto rows = [&](int f0, int f1) {
        if (f1 <= f0) return;
        GemvArgs g;
        g.a = k->blocks.p + static_cast<size_t>(f0) * mpf * mpf * nb;
        g.x = x;
        g.y = y + static_cast<size_t>(f0) * mpf;
        g.rows = mpf;
        g.cols = mpf * nb;
        g.batch = f1 - f0;
        g.idx = k->nbr32.p + static_cast<size_t>(f0) * nb;
        g.width = mpf;
        g.comp = 1;
        launch_team_gemv(c, g);
    };
    if (c->comm && tuning().overlap_halo && k->nf_interior > 0) {
        c->comm->halo_begin(c, const_cast<double*>(x), mpf);
        rows(0, k->nf_interior);
        c->comm->halo_end(c);
        rows(k->nf_interior, k->nf);
        return;
    }
    if (c->comm) c->comm->halo(c, const_cast<double*>(x), mpf);
    rows(0, k->nf);
}

void apply_base_device(hdgb_precond* p, const double* y, double* z, const PolyEpi* epi) {
    hdgb_ctx* c = p->ctx;
    const int64_t n = static_cast<int64_t>(p->mpf) * p->nf;
    switch (p->kind) {
        case HDGB_PC_IDENTITY:
            if (epi) launch_poly_update(c, *epi, y, n);
            else if (y != z) HDGB_CUDA(cudaMemcpyAsync(z, y, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
            break;
        case HDGB_PC_BJ: {
            // apply_bj (preconditioner.cpp:48-52)
            GemvArgs g;
            g.a = p->bj_inv.p; g.x = y; g.y = z;
            g.rows = p->mpf; g.cols = p->mpf; g.batch = p->nf;
            launch_team_gemv(c, g);
            if (epi) launch_poly_update(c, *epi, z, n);  // both recurrence updates in one pass over t
            break;
        }
        default: {
            // apply_asm (preconditioner.cpp:86-105): gather_element_trace fused into the element
            // solve, then the scatter-add written as an atomics-free face gather (side 0 first).
            const DiscView& v = p->disc->view;
            // domain decomposition: ghost elements are solved redundantly, so y is needed on every
            // local face; a shared face then finds both sides' corrections locally.  Elements whose faces
            // are all owned (ne_interior, numbered first) are solved while the halo exchange is in flight.
            auto elems = [&](int e0, int e1) {
                if (e1 <= e0) return;
                GemvArgs g;
                g.a = p->asm_inv.p + static_cast<size_t>(e0) * v.nfl * v.nfl;
                g.x = y;
                g.y = p->ze.p + static_cast<size_t>(e0) * v.nfl;
                g.rows = v.nfl; g.cols = v.nfl; g.batch = e1 - e0;
                g.idx = v.elem_faces + static_cast<size_t>(e0) * v.n_lfe;
                g.width = v.mpf; g.comp = 1;
                launch_team_gemv(c, g);
            };
            const int ni = p->disc->ne_interior;
            if (c->comm && tuning().overlap_halo && ni > 0) {
                c->comm->halo_begin(c, const_cast<double*>(y), v.mpf);
                elems(0, ni);
                c->comm->halo_end(c);
                elems(ni, v.ne);
            } else {
                if (c->comm) c->comm->halo(c, const_cast<double*>(y), v.mpf);
                elems(0, v.ne);
            }
            // the polynomial recurrence updates ride on the face sum (the value t is never stored)
            launch_face_sum(c, p->ze.p, v.face_elems, v.face_lidx, v.nf_owned, v.mpf, v.n_lfe, z,
                            p->kind == HDGB_PC_RAS ? 1 : 2, epi);
            break;
        }
    }
}

// apply_poly (preconditioner.cpp:246-283); op = v -> base(K v).
void apply_poly_op(hdgb_precond* p, const DevOp& base, hdgb_matrix* k, const double* y, double* z) {
    hdgb_ctx* c = p->ctx;
    const int64_t n = k->n_dof();
    const size_t ld = static_cast<size_t>(k->n_local());
    if (p->wq.n != ld) { p->wq.alloc(ld); p->wt.alloc(ld); p->ws.alloc(ld); p->wkv.alloc(ld); }
    double *q = p->wq.p, *t = p->wt.p, *s = p->ws.p, *kv = p->wkv.p;
    double* w = z;
    base(y, q);
    launch_fill(c, w, 0.0, n);
    auto op = [&](const double* in, double* out) {
        matvec_device(k, in, kv);
        base(kv, out);
        ++p->inner_ops;
    };
    const size_t cnt = p->ritz.size() / 2;
    size_t i = 0;
    while (i < cnt) {
        const double re = p->ritz[2 * i], im = p->ritz[2 * i + 1];
        if (im == 0.0) {
            const double inv = 1.0 / re;
            launch_axpby(c, inv, q, 1.0, w, n);   // w += inv q
            op(q, t);
            launch_axpby(c, -inv, t, 1.0, q, n);  // q -= inv t
            i += 1;
        } else {
            const double inv = 1.0 / (re * re + im * im);
            op(q, t);
            launch_poly_pair_mid(c, 2.0 * re, inv, q, t, s, w, n);  // s = 2a q - t ; w += inv s
            op(s, t);
            launch_axpby(c, -inv, t, 1.0, q, n);
            i += 2;
        }
    }
}

// apply_poly (preconditioner.cpp:246-283) with the preconditioner's own base: identical recurrence, the vector
// updates w += q / theta, q -= t / theta (and the pair step) applied inside the kernel that produces t.
void apply_poly_fused(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z) {
    hdgb_ctx* c = p->ctx;
    const int64_t n = k->n_dof();
    const size_t ld = static_cast<size_t>(k->n_local());
    if (p->wq.n != ld) { p->wq.alloc(ld); p->wt.alloc(ld); p->ws.alloc(ld); p->wkv.alloc(ld); }
    double *q = p->wq.p, *t = p->wt.p, *s = p->ws.p, *kv = p->wkv.p;
    double* w = z;
    apply_base_device(p, y, q);
    launch_fill(c, w, 0.0, n);
    auto op = [&](const double* in, const PolyEpi& e) {
        matvec_device(k, in, kv);
        apply_base_device(p, kv, t, &e);
        ++p->inner_ops;
    };
    const size_t cnt = p->ritz.size() / 2;
    size_t i = 0;
    while (i < cnt) {
        const double re = p->ritz[2 * i], im = p->ritz[2 * i + 1];
        PolyEpi e;
        e.q = q; e.w = w; e.s = s;
        if (im == 0.0) {
            e.mode = PolyEpi::kReal;
            e.a = 1.0 / re;
            op(q, e);  // w += q / theta ; q -= op(q) / theta
            i += 1;
        } else {
            const double inv = 1.0 / (re * re + im * im);
            e.mode = PolyEpi::kMid;
            e.a = 2.0 * re;
            e.b = inv;
            op(q, e);  // s = 2a q - op(q) ; w += inv s
            e.mode = PolyEpi::kLast;
            e.a = inv;
            op(s, e);  // q -= inv op(s)
            i += 2;
        }
    }
}

static void apply_poly_device(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z) {
    if (tuning().poly_fused) apply_poly_fused(p, k, y, z);
    else apply_poly_op(p, [p](const double* in, double* out) { apply_base_device(p, in, out); }, k, y, z);
}

void apply_precond_device(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z) {
    if (!p) {
        if (y != z)
            HDGB_CUDA(cudaMemcpyAsync(z, y, k->n_dof() * sizeof(double), cudaMemcpyDeviceToDevice, k->ctx->stream));
        return;
    }
    if (p->poly_degree == 0 || p->ritz.empty()) apply_base_device(p, y, z);
    else apply_poly_device(p, k, y, z);
}

// compute_harmonic_ritz (preconditioner.cpp:119-205): seeded start vector, MGS Arnoldi on the
// device, small eigen-solve and Leja ordering on the host.
std::vector<std::complex<double>> harmonic_ritz_op(hdgb_ctx* c, const DevOp& op, int64_t n, int64_t ld, int degree,
                                                   uint64_t seed, const int64_t* face_gid, int nf_local, int mpf,
                                                   int64_t n_global, bool* breakdown_out) {
    if (degree < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: polynomial degree must be >= 1");
    // Seeded start vector over the GLOBAL unknowns (preconditioner.cpp:128-132); a rank keeps the
    // entries of its local faces, so the sequence does not depend on the partition.
    if (degree > n_global) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: polynomial degree exceeds the operator dimension");
    std::mt19937_64 rng(seed);
    std::vector<double> vg(n_global);
    for (double& x : vg) x = 2.0 * (static_cast<double>(rng() >> 11) * 0x1p-53) - 1.0;
    double acc = 0.0;
    for (double x : vg) acc += x * x;  // same ascending order as the reference's dot
    const double nv = std::sqrt(acc);
    std::vector<double> v0(ld, 0.0);
    if (!face_gid) {
        for (int64_t i = 0; i < n; ++i) v0[i] = vg[i] / nv;
    } else {
        for (int f = 0; f < nf_local; ++f) {
            const int64_t gf = face_gid[f];
            for (int r = 0; r < mpf; ++r) v0[static_cast<int64_t>(f) * mpf + r] = vg[gf * mpf + r] / nv;
        }
    }

    const int pmax = degree;
    DevBuf<double> basis(static_cast<size_t>(pmax) * ld), w(ld), sc(pmax + 4);
    DevBuf<double> partial(multi_dot_workspace_doubles(n, 1));
    HDGB_CUDA(cudaMemcpyAsync(basis.p, v0.data(), ld * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    std::vector<double> hess(static_cast<size_t>(pmax + 1) * pmax, 0.0);
    auto h = [&](int i, int j) -> double& { return hess[static_cast<size_t>(j) * (pmax + 1) + i]; };
    auto fetch = [&](const double* dev) {
        double v;
        HDGB_CUDA(cudaMemcpyAsync(&v, dev, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        return v;
    };
    auto reduce = [&](double* dev, int cnt) { if (c->comm) c->comm->allreduce(c, dev, cnt); };
    int p_eff = 0;
    double scale = 1.0;
    std::vector<double> col(pmax + 2);
    for (int j = 0; j < pmax; ++j) {
        op(basis.p + static_cast<size_t>(j) * ld, w.p);
        if (j == 0) {
            launch_sumsq(c, w.p, n, sc.p, partial.p);
            reduce(sc.p, 1);
            scale = std::max(1.0, std::sqrt(fetch(sc.p)));
        }
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt (preconditioner.cpp:146-150)
            const double* vi = basis.p + static_cast<size_t>(i) * ld;
            launch_multi_dot(c, vi, ld, 1, w.p, n, sc.p + i, partial.p);
            reduce(sc.p + i, 1);
            launch_multi_axpy(c, vi, ld, 1, sc.p + i, -1.0, w.p, n, nullptr, partial.p);
        }
        launch_sumsq(c, w.p, n, sc.p + j + 1, partial.p);
        reduce(sc.p + j + 1, 1);
        HDGB_CUDA(cudaMemcpyAsync(col.data(), sc.p, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        for (int i = 0; i <= j; ++i) h(i, j) = col[i];
        const double hn = std::sqrt(col[j + 1]);
        h(j + 1, j) = hn;
        p_eff = j + 1;
        if (!std::isfinite(hn)) throw Failure(HDGB_ERR_NAN_DETECTED, "NaN detected in harmonic Ritz Arnoldi");
        if (hn < 1e-14 * scale) break;
        if (j + 1 < pmax) launch_scale_dev(c, w.p, sc.p + j + 1, 0, basis.p + static_cast<size_t>(j + 1) * ld, n);
    }
    HDGB_CUDA(cudaStreamSynchronize(c->stream));
    if (breakdown_out) *breakdown_out = p_eff < pmax;
    return harmonic_ritz_from_hessenberg(hess.data(), pmax, p_eff);
}

static std::vector<std::complex<double>> harmonic_ritz_device(hdgb_precond* p, hdgb_matrix* k, int degree,
                                                              uint64_t seed, bool* breakdown_out) {
    const int64_t n = k->n_dof(), ld = k->n_local();
    const bool dd = p->disc && !p->disc->face_gid.empty();
    DevBuf<double> kv(ld);
    return harmonic_ritz_op(p->ctx, [&](const double* in, double* out) {
                                matvec_device(k, in, kv.p);
                                apply_base_device(p, kv.p, out);
                            },
                            n, ld, degree, seed, dd ? p->disc->face_gid.data() : nullptr, k->nf_local, k->mpf(),
                            dd ? p->disc->nf_global * k->mpf() : n, breakdown_out);
}

// Chebyshev nodes of the real interval covering the Ritz estimates, Leja-ordered.
static std::vector<std::complex<double>> chebyshev_nodes(const std::vector<std::complex<double>>& ritz, int degree) {
    double lo = INFINITY, hi = -INFINITY;
    for (const auto& t : ritz) {
        lo = std::min(lo, t.real());
        hi = std::max(hi, t.real());
    }
    if (!(lo > 0.0)) lo = hi / 30.0;  // indefinite / tiny estimate: fall back to a fixed ratio
    if (hi <= lo) hi = lo * (1.0 + 1e-8);
    const double kPi = 3.14159265358979323846;
    std::vector<std::complex<double>> nodes;
    for (int j = 0; j < degree; ++j) {
        const double x = std::cos(kPi * (2.0 * j + 1.0) / (2.0 * degree));
        nodes.emplace_back(0.5 * (hi + lo) + 0.5 * (hi - lo) * x, 0.0);
    }
    return leja_order(nodes);
}

static std::unique_ptr<hdgb_precond> new_precond(hdgb_ctx* c, int kind, int mpf, int nf, int nf_local, int n_lfe, hdgb_disc* d) {
    std::unique_ptr<hdgb_precond> p(new hdgb_precond());
    p->ctx = c;
    p->kind = kind;
    p->mpf = mpf;
    p->nf = nf;
    p->nf_local = nf_local;
    p->n_lfe = n_lfe;
    p->disc = d;
    return p;
}

// build_bj (preconditioner.cpp:30-46)
hdgb_precond* build_bj_device(hdgb_matrix* k) {
    hdgb_ctx* c = k->ctx;
    auto p = new_precond(c, HDGB_PC_BJ, k->mpf(), k->nf, k->nf_local, k->n_lfe, nullptr);
    const int mpf = p->mpf;
    p->bj_inv.alloc(static_cast<size_t>(mpf) * mpf * k->nf);
    launch_extract_diag(c, k->blocks.p, k->nf, mpf, k->nb(), p->bj_inv.p);
    device_lu_invert(c, mpf, k->nf, p->bj_inv.p, p->bj_inv.p, "build_bj (face block)", HDGB_ERR_SINGULAR_BLOCK);
    return p.release();
}

// build_asm (preconditioner.cpp:54-84).  The enriched diagonal sub-block of a face (both sides' K-bar_ll summed,
// side 0 first, :59-75) IS the face's self block K_ff of the assembled operator: diag_from_k (mpf^2 per local
// face, owned part filled) passes it in when K exists; nullptr sums it from K-bar directly, as the reference does.
// Halo faces receive theirs from the owner, so ghost elements are enriched without a second ghost layer.
hdgb_precond* build_asm_device(const hdgb_ops* o, hdgb_disc* d, int kind, const double* diag_from_k) {
    if (!o || !d) throw Failure(HDGB_ERR_GENERIC, "build_asm needs the element operators and the discretisation");
    hdgb_ctx* c = d->ctx;
    const DiscView& v = d->view;
    if (o->ne != v.ne || o->nfl != v.nfl) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: build_asm operators / mesh");
    auto p = new_precond(c, kind, v.mpf, v.nf_owned, v.nf, v.n_lfe, d);
    p->ne = v.ne;
    p->asm_inv.alloc(static_cast<size_t>(v.nfl) * v.nfl * v.ne);
    DevBuf<double> diag;
    double* dg = const_cast<double*>(diag_from_k);
    if (!dg) {
        diag.alloc(static_cast<size_t>(v.mpf) * v.mpf * v.nf);
        launch_face_diag(c, v, o->kbar.p, diag.p);
        dg = diag.p;
    }
    if (c->comm) c->comm->halo(c, dg, v.mpf * v.mpf);
    launch_asm_enrich(c, v, o->kbar.p, dg, p->asm_inv.p);
    device_lu_invert(c, v.nfl, v.ne, p->asm_inv.p, p->asm_inv.p, "build_asm (element block)", HDGB_ERR_SINGULAR_BLOCK);
    p->ze.alloc(static_cast<size_t>(v.nfl) * v.ne);
    return p.release();
}

hdgb_precond* build_preconditioner_spec(hdgb_matrix* k, const hdgb_ops* o, hdgb_disc* d, const hdgb_precond_spec& spec) {
    hdgb_ctx* c = k->ctx;
    std::unique_ptr<hdgb_precond> p;
    const int64_t n = k->n_dof();
    switch (spec.kind) {
        case HDGB_PC_IDENTITY: p = new_precond(c, HDGB_PC_IDENTITY, k->mpf(), k->nf, k->nf_local, k->n_lfe, d); break;
        case HDGB_PC_BJ:
            p.reset(build_bj_device(k));
            p->disc = d;
            break;
        case HDGB_PC_ASM:
        case HDGB_PC_RAS: {
            if (!o || !d) throw Failure(HDGB_ERR_GENERIC, "build_asm needs the element operators and the discretisation");
            if (d->view.mpf != k->mpf() || d->view.nf_owned != k->nf)
                throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: build_asm matrix / mesh");
            DevBuf<double> diag(static_cast<size_t>(k->mpf()) * k->mpf() * d->view.nf);
            launch_extract_diag(c, k->blocks.p, k->nf, k->mpf(), k->nb(), diag.p);
            p.reset(build_asm_device(o, d, spec.kind, diag.p));
            break;
        }
        default: throw Failure(HDGB_ERR_UNSUPPORTED, "unknown preconditioner kind");
    }
    if (spec.poly_degree > 0) {
        const int degree = static_cast<int>(std::min<int64_t>(spec.poly_degree, n));  // newton.cpp:41
        const int64_t ld = k->n_local();
        p->wq.alloc(ld); p->wt.alloc(ld); p->ws.alloc(ld); p->wkv.alloc(ld);
        bool breakdown = false;
        std::vector<std::complex<double>> th = harmonic_ritz_device(p.get(), k, degree, spec.ritz_seed, &breakdown);
        p->poly_kind = spec.poly_kind;
        if (spec.poly_kind == HDGB_POLY_CHEBYSHEV && !th.empty()) th = chebyshev_nodes(th, degree);
        p->ritz.clear();
        for (const auto& t : th) { p->ritz.push_back(t.real()); p->ritz.push_back(t.imag()); }
        p->poly_degree = degree;
    }
    return p.release();
}

hdgb_matrix* assemble_global_device(hdgb_disc* d, const hdgb_ops* o) {
    hdgb_ctx* c = d->ctx;
    const DiscView& v = d->view;
    std::unique_ptr<hdgb_matrix> k(new hdgb_matrix());
    k->ctx = c;
    k->m = v.M;  // the reference leaves m = 1 (face_matrix.hpp:27); identical for its scalar models
    k->pf = v.pf;
    k->n_lfe = v.n_lfe;
    k->nf = v.nf_owned;   // rows: owned faces (both adjacent elements are local)
    k->nf_local = v.nf;   // vectors: all local faces
    k->nf_interior = d->nf_interior;
    const size_t row = static_cast<size_t>(v.mpf) * v.mpf * k->nb();
    k->blocks.alloc(row * k->nf);
    k->rhs.alloc(static_cast<size_t>(v.mpf) * v.nf);
    k->rhs.zero(c->stream);
    k->nbr32.alloc(static_cast<size_t>(k->nf) * k->nb());
    DiscView rows = v;
    rows.nf = k->nf;
    launch_fill_neighbors(c, rows, k->nbr32.p);
    launch_assemble_global(c, rows, o->kbar.p, o->rbar.p, k->blocks.p, k->rhs.p);
    return k.release();
}

static void ensure_host_neighbors(hdgb_matrix* k) {
    if (k->neighbor_valid) return;
    std::vector<int> h = k->nbr32.to_host(k->ctx->stream);
    k->neighbor.resize(h.size());
    for (size_t i = 0; i < h.size(); ++i) k->neighbor[i] = h[i];  // kNoFace = -1 widens unchanged
    k->neighbor_valid = true;
}

}  // namespace hdgb

extern "C" {

void hdgb_precond_spec_default(hdgb_precond_spec* s) {
    s->kind = HDGB_PC_BJ;
    s->poly_degree = 0;
    s->ritz_seed = 12345;
    s->ritz_per_restart = 0;
    s->poly_kind = HDGB_POLY_GMRES;
}

hdgb_status hdgb_assemble_global(hdgb_disc* d, const hdgb_ops* o, hdgb_matrix** out, double* rhs) {
    *out = nullptr;
    hdgb_ctx* c = d->ctx;
    return guarded(c, [&] {
        if (o->ne != d->view.ne || o->nfl != d->view.nfl)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: assemble_global operators / mesh");
        std::unique_ptr<hdgb_matrix> k(assemble_global_device(d, o));
        if (rhs) HDGB_CUDA(cudaMemcpyAsync(rhs, k->rhs.p, k->rhs.n * sizeof(double), cudaMemcpyDefault, c->stream));
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        *out = k.release();
    });
}

hdgb_status hdgb_matrix_create(hdgb_ctx* c, int m, int pf, int n_lfe, int nf, const int64_t* neighbor,
                               const double* blocks, hdgb_matrix** out) {
    *out = nullptr;
    return guarded(c, [&] {
        if (m < 1 || pf < 1 || n_lfe < 1 || nf < 0)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: invalid face-block matrix dimensions");
        std::unique_ptr<hdgb_matrix> k(new hdgb_matrix());
        k->ctx = c; k->m = m; k->pf = pf; k->n_lfe = n_lfe; k->nf = nf; k->nf_local = nf;
        const size_t nn = static_cast<size_t>(nf) * k->nb();
        k->neighbor.assign(neighbor, neighbor + nn);
        std::vector<int> h32(nn);
        for (size_t i = 0; i < nn; ++i) {
            const int64_t g = neighbor[i];
            if (g < -1 || g >= nf) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: neighbour id out of range", static_cast<int64_t>(i / k->nb()));
            h32[i] = static_cast<int>(g);
        }
        k->neighbor_valid = true;
        k->nbr32.from_host(h32, c->stream);
        const size_t total = static_cast<size_t>(k->mpf()) * k->mpf() * k->nb() * nf;
        k->blocks.alloc(total);
        if (blocks) HDGB_CUDA(cudaMemcpyAsync(k->blocks.p, blocks, total * sizeof(double), cudaMemcpyDefault, c->stream));
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        *out = k.release();
    });
}

void hdgb_matrix_destroy(hdgb_matrix* k) { delete k; }

hdgb_status hdgb_matrix_dims(const hdgb_matrix* k, int* out4) {
    out4[0] = k->m; out4[1] = k->pf; out4[2] = k->n_lfe; out4[3] = k->nf;
    return HDGB_OK;
}

hdgb_status hdgb_matrix_get_neighbor(const hdgb_matrix* kc, int64_t* out) {
    hdgb_matrix* k = const_cast<hdgb_matrix*>(kc);
    return guarded(k->ctx, [&] {
        ensure_host_neighbors(k);
        std::memcpy(out, k->neighbor.data(), k->neighbor.size() * sizeof(int64_t));
    });
}

hdgb_status hdgb_matrix_get_blocks(const hdgb_matrix* k, double* out) {
    return guarded(k->ctx, [&] {
        HDGB_CUDA(cudaMemcpyAsync(out, k->blocks.p, k->blocks.n * sizeof(double), cudaMemcpyDefault, k->ctx->stream));
        HDGB_CUDA(cudaStreamSynchronize(k->ctx->stream));
    });
}

double* hdgb_matrix_blocks_ptr(hdgb_matrix* k) { return k->blocks.p; }
double* hdgb_matrix_rhs(hdgb_matrix* k) { return k->rhs.p; }

hdgb_status hdgb_block_matvec(hdgb_matrix* k, const double* x, double* y) {
    hdgb_ctx* c = k->ctx;
    return guarded(c, [&] {
        const size_t n = k->n_local();
        InArg X(c, x, n);
        OutArg Y(c, y, n);
        matvec_device(k, X.dev, Y.dev);
        Y.commit();
        if (!X.tmp.p && !Y.host) return;  // fully device-resident call stays asynchronous
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_gather_extended(hdgb_matrix* k, const double* x, double* out) {
    hdgb_ctx* c = k->ctx;
    return guarded(c, [&] {
        const size_t n = k->n_dof();
        InArg X(c, x, n);
        OutArg Y(c, out, n * k->nb());
        launch_gather_extended(c, X.dev, k->nbr32.p, k->nf, k->nb(), k->mpf(), Y.dev);
        Y.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_matrix_write(hdgb_matrix* k, const double* rhs, const char* path) {
    hdgb_ctx* c = k->ctx;
    return guarded(c, [&] {
        ensure_host_neighbors(k);
        std::vector<double> blocks = k->blocks.to_host(c->stream);
        std::vector<double> r(k->n_dof(), 0.0);
        const double* src = rhs ? rhs : k->rhs.p;
        if (src) {
            HDGB_CUDA(cudaMemcpyAsync(r.data(), src, r.size() * sizeof(double), cudaMemcpyDefault, c->stream));
            HDGB_CUDA(cudaStreamSynchronize(c->stream));
        }
        const std::string p = path;
        std::FILE* fp = std::fopen(path, "wb");
        if (!fp) throw Failure(HDGB_ERR_IO, "cannot open " + p + " for writing");
        const uint32_t header[5] = {1u, static_cast<uint32_t>(k->m), static_cast<uint32_t>(k->pf),
                                    static_cast<uint32_t>(k->n_lfe), static_cast<uint32_t>(k->nf)};
        bool ok = std::fwrite("HDGK", 1, 4, fp) == 4;
        ok = ok && std::fwrite(header, 1, sizeof(header), fp) == sizeof(header);
        ok = ok && std::fwrite(k->neighbor.data(), sizeof(int64_t), k->neighbor.size(), fp) == k->neighbor.size();
        ok = ok && std::fwrite(blocks.data(), sizeof(double), blocks.size(), fp) == blocks.size();
        ok = ok && std::fwrite(r.data(), sizeof(double), r.size(), fp) == r.size();
        std::fclose(fp);
        if (!ok) throw Failure(HDGB_ERR_IO, "short write to " + p);
    });
}

hdgb_status hdgb_matrix_read(hdgb_ctx* c, const char* path, hdgb_matrix** out, double* rhs) {
    *out = nullptr;
    return guarded(c, [&] {
        const std::string p = path;
        std::FILE* fp = std::fopen(path, "rb");
        if (!fp) throw Failure(HDGB_ERR_IO, "cannot open " + p);
        struct Closer { std::FILE* f; ~Closer() { std::fclose(f); } } closer{fp};
        char magic[4];
        if (std::fread(magic, 1, 4, fp) != 4) throw Failure(HDGB_ERR_IO, "short read from " + p);
        if (std::memcmp(magic, "HDGK", 4) != 0) throw Failure(HDGB_ERR_IO, p + " is not a matrix dump");
        uint32_t header[5];
        if (std::fread(header, 1, sizeof(header), fp) != sizeof(header)) throw Failure(HDGB_ERR_IO, "short read from " + p);
        if (header[0] != 1u) throw Failure(HDGB_ERR_IO, p + ": unsupported format version");
        const int m = static_cast<int>(header[1]), pf = static_cast<int>(header[2]);
        const int n_lfe = static_cast<int>(header[3]), nf = static_cast<int>(header[4]);
        const int nb = 2 * n_lfe - 1;
        std::vector<int64_t> nbr(static_cast<size_t>(nf) * nb);
        if (std::fread(nbr.data(), sizeof(int64_t), nbr.size(), fp) != nbr.size()) throw Failure(HDGB_ERR_IO, "short read from " + p);
        std::vector<double> blocks(static_cast<size_t>(m) * pf * m * pf * nb * nf);
        if (std::fread(blocks.data(), sizeof(double), blocks.size(), fp) != blocks.size()) throw Failure(HDGB_ERR_IO, "short read from " + p);
        std::vector<double> r(static_cast<size_t>(m) * pf * nf);
        if (std::fread(r.data(), sizeof(double), r.size(), fp) != r.size()) throw Failure(HDGB_ERR_IO, "short read from " + p);
        hdgb_matrix* k = nullptr;
        hdgb_status st = hdgb_matrix_create(c, m, pf, n_lfe, nf, nbr.data(), blocks.data(), &k);
        if (st != HDGB_OK) throw Failure(st, c->err, c->err_index);
        k->rhs.alloc(r.size());
        k->rhs.upload(r.data(), r.size(), c->stream);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        if (rhs) std::memcpy(rhs, r.data(), r.size() * sizeof(double));
        *out = k;
    });
}

// ---- preconditioners -----------------------------------------------------------------------------------
hdgb_status hdgb_build_preconditioner(hdgb_matrix* k, const hdgb_ops* o, hdgb_disc* d, const hdgb_precond_spec* spec,
                                      hdgb_precond** out) {
    *out = nullptr;
    return guarded(k->ctx, [&] {
        hdgb_precond_spec s;
        hdgb_precond_spec_default(&s);
        if (spec) s = *spec;
        *out = build_preconditioner_spec(k, o, d, s);
        HDGB_CUDA(cudaStreamSynchronize(k->ctx->stream));
    });
}

void hdgb_precond_destroy(hdgb_precond* p) { delete p; }

hdgb_status hdgb_precond_get(const hdgb_precond* p, const char* name, double* dst, int64_t cap, int64_t* n) {
    return guarded(p->ctx, [&] {
        const std::string s = name;
        if (s == "ritz") {
            if (n) *n = static_cast<int64_t>(p->ritz.size());
            if (dst) {
                if (cap < static_cast<int64_t>(p->ritz.size())) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "destination too small");
                std::memcpy(dst, p->ritz.data(), p->ritz.size() * sizeof(double));
            }
            return;
        }
        const DevBuf<double>* b = nullptr;
        if (s == "bj_inv") b = &p->bj_inv;
        else if (s == "asm_inv") b = &p->asm_inv;
        else throw Failure(HDGB_ERR_GENERIC, "unknown preconditioner field " + s);
        if (n) *n = static_cast<int64_t>(b->n);
        if (dst) {
            if (cap < static_cast<int64_t>(b->n)) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "destination too small");
            HDGB_CUDA(cudaMemcpyAsync(dst, b->p, b->n * sizeof(double), cudaMemcpyDeviceToHost, p->ctx->stream));
            HDGB_CUDA(cudaStreamSynchronize(p->ctx->stream));
        }
    });
}

hdgb_status hdgb_precond_set_ritz(hdgb_precond* p, const double* reim, int count) {
    return guarded(p->ctx, [&] {
        p->ritz.assign(reim, reim + 2 * static_cast<size_t>(count));
        p->poly_degree = count;
        const size_t n = static_cast<size_t>(p->mpf) * std::max(p->nf, p->nf_local);
        if (count > 0 && p->wq.n != n) { p->wq.alloc(n); p->wt.alloc(n); p->ws.alloc(n); p->wkv.alloc(n); }
    });
}

hdgb_status hdgb_precond_apply_base(hdgb_precond* p, const double* y, double* z) {
    hdgb_ctx* c = p->ctx;
    return guarded(c, [&] {
        const size_t n = static_cast<size_t>(p->mpf) * std::max(p->nf, p->nf_local);
        InArg Y(c, y, n);
        OutArg Z(c, z, n);
        apply_base_device(p, Y.dev, Z.dev);
        Z.commit();
        if (!Y.tmp.p && !Z.host) return;
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_precond_apply(hdgb_precond* p, hdgb_matrix* k, const double* y, double* z) {
    hdgb_ctx* c = p->ctx;
    return guarded(c, [&] {
        const size_t n = static_cast<size_t>(p->mpf) * std::max(p->nf, p->nf_local);
        InArg Y(c, y, n);
        OutArg Z(c, z, n);
        apply_precond_device(p, k, Y.dev, Z.dev);
        Z.commit();
        if (!Y.tmp.p && !Z.host) return;
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

// ---- per-function entry points of preconditioner.hpp:31-76 ------------------------------------------------
hdgb_status hdgb_build_bj(hdgb_matrix* k, hdgb_precond** out) {
    *out = nullptr;
    return guarded(k->ctx, [&] {
        *out = build_bj_device(k);
        HDGB_CUDA(cudaStreamSynchronize(k->ctx->stream));
    });
}

hdgb_status hdgb_build_asm(const hdgb_ops* o, hdgb_disc* d, hdgb_precond** out) {
    *out = nullptr;
    return guarded(d->ctx, [&] {
        *out = build_asm_device(o, d, HDGB_PC_ASM, nullptr);
        HDGB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    });
}

static hdgb_status apply_kind(hdgb_precond* p, int kind_a, int kind_b, const char* what, const double* y, double* z) {
    hdgb_ctx* c = p->ctx;
    return guarded(c, [&] {
        if (p->kind != kind_a && p->kind != kind_b)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, std::string("dimension mismatch: ") + what + " on a preconditioner of another kind");
        const size_t n = static_cast<size_t>(p->mpf) * std::max(p->nf, p->nf_local);
        InArg Y(c, y, n);
        OutArg Z(c, z, n);
        apply_base_device(p, Y.dev, Z.dev);
        Z.commit();
        if (!Y.tmp.p && !Z.host) return;
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_apply_bj(hdgb_precond* p, const double* y, double* z) { return apply_kind(p, HDGB_PC_BJ, HDGB_PC_BJ, "apply_bj", y, z); }
hdgb_status hdgb_apply_asm(hdgb_precond* p, const double* y, double* z) { return apply_kind(p, HDGB_PC_ASM, HDGB_PC_RAS, "apply_asm", y, z); }

hdgb_status hdgb_precond_create(hdgb_ctx* c, int kind, int mpf, int nf, hdgb_disc* d, const double* inv,
                                const double* ritz_reim, int n_ritz, hdgb_precond** out) {
    *out = nullptr;
    return guarded(c, [&] {
        if (mpf < 1 || nf < 0 || n_ritz < 0) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: invalid preconditioner dimensions");
        std::unique_ptr<hdgb_precond> p;
        switch (kind) {
            case HDGB_PC_IDENTITY: p = new_precond(c, kind, mpf, nf, nf, 0, d); break;
            case HDGB_PC_BJ: {
                if (!inv) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: block-Jacobi inverses missing");
                p = new_precond(c, kind, mpf, nf, nf, 0, d);
                p->bj_inv.alloc(static_cast<size_t>(mpf) * mpf * nf);
                HDGB_CUDA(cudaMemcpyAsync(p->bj_inv.p, inv, p->bj_inv.n * sizeof(double), cudaMemcpyDefault, c->stream));
                break;
            }
            case HDGB_PC_ASM:
            case HDGB_PC_RAS: {
                if (!inv || !d) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: additive Schwarz needs the inverses and the discretisation");
                const DiscView& v = d->view;
                if (v.mpf != mpf || v.nf_owned != nf) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: preconditioner / mesh");
                p = new_precond(c, kind, mpf, v.nf_owned, v.nf, v.n_lfe, d);
                p->ne = v.ne;
                p->asm_inv.alloc(static_cast<size_t>(v.nfl) * v.nfl * v.ne);
                HDGB_CUDA(cudaMemcpyAsync(p->asm_inv.p, inv, p->asm_inv.n * sizeof(double), cudaMemcpyDefault, c->stream));
                p->ze.alloc(static_cast<size_t>(v.nfl) * v.ne);
                break;
            }
            default: throw Failure(HDGB_ERR_UNSUPPORTED, "unknown preconditioner kind");
        }
        if (n_ritz > 0) {
            p->ritz.assign(ritz_reim, ritz_reim + 2 * static_cast<size_t>(n_ritz));
            p->poly_degree = n_ritz;
        }
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        *out = p.release();
    });
}

// Wraps a C callback as a device operator; a non-zero return aborts the calling algorithm.
static DevOp wrap_op(hdgb_op_fn fn, void* user, int64_t n, const char* what) {
    return [fn, user, n, what](const double* in, double* out) {
        if (fn(user, in, out, n) != 0) throw Failure(HDGB_ERR_GENERIC, std::string(what) + ": operator callback failed");
    };
}

hdgb_status hdgb_compute_harmonic_ritz(hdgb_ctx* c, hdgb_op_fn op, void* user, int64_t n_dof, int degree, uint64_t seed,
                                       double* out_reim, int* n_out) {
    if (n_out) *n_out = 0;
    return guarded(c, [&] {
        if (!op) throw Failure(HDGB_ERR_GENERIC, "compute_harmonic_ritz: operator callback missing");
        const auto th = harmonic_ritz_op(c, wrap_op(op, user, n_dof, "compute_harmonic_ritz"), n_dof, n_dof, degree, seed,
                                         nullptr, 0, 1, n_dof, nullptr);
        for (size_t i = 0; i < th.size(); ++i) { out_reim[2 * i] = th[i].real(); out_reim[2 * i + 1] = th[i].imag(); }
        if (n_out) *n_out = static_cast<int>(th.size());
    });
}

hdgb_status hdgb_apply_poly(hdgb_precond* p, hdgb_op_fn base_apply, void* user, hdgb_matrix* k, const double* y, double* z,
                            int64_t* inner_ops) {
    hdgb_ctx* c = p->ctx;
    return guarded(c, [&] {
        if (static_cast<int64_t>(p->mpf) * p->nf != k->n_dof())
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: preconditioner / operator size");
        const size_t n = static_cast<size_t>(k->n_local());
        InArg Y(c, y, n);
        OutArg Z(c, z, n);
        const int64_t before = p->inner_ops;
        if (base_apply) apply_poly_op(p, wrap_op(base_apply, user, k->n_dof(), "apply_poly"), k, Y.dev, Z.dev);
        else apply_poly_op(p, [p](const double* in, double* out) { apply_base_device(p, in, out); }, k, Y.dev, Z.dev);
        if (inner_ops) *inner_ops += p->inner_ops - before;
        Z.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int64_t hdgb_precond_inner_ops(const hdgb_precond* p) { return p->inner_ops; }

hdgb_status hdgb_leja_order(const double* reim, int n, double* out_reim, int* n_out) {
    try {
        std::vector<std::complex<double>> th(n);
        for (int i = 0; i < n; ++i) th[i] = {reim[2 * i], reim[2 * i + 1]};
        const auto o = leja_order(th);
        for (size_t i = 0; i < o.size(); ++i) { out_reim[2 * i] = o[i].real(); out_reim[2 * i + 1] = o[i].imag(); }
        *n_out = static_cast<int>(o.size());
        return HDGB_OK;
    } catch (...) {
        return HDGB_ERR_GENERIC;
    }
}

hdgb_status hdgb_harmonic_ritz_from_hessenberg(const double* hess, int pmax, int p_eff, double* out_reim, int* n_out) {
    try {
        const auto o = harmonic_ritz_from_hessenberg(hess, pmax, p_eff);
        for (size_t i = 0; i < o.size(); ++i) { out_reim[2 * i] = o[i].real(); out_reim[2 * i + 1] = o[i].imag(); }
        *n_out = static_cast<int>(o.size());
        return HDGB_OK;
    } catch (...) {
        return HDGB_ERR_GENERIC;
    }
}

}  // extern "C"
