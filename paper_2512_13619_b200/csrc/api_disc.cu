// C ABI: discretisation handle, PDE model, state, and the element-local operators (A3-A6).
#include <cmath>
#include <cstring>

#include "solver.cuh"

using namespace hdgb;

namespace {

template <class T>
void upload(hdgb_ctx* c, DevBuf<T>& dst, const std::vector<T>& src) {
    dst.alloc(src.size());
    if (!src.empty())
        HDGB_CUDA(cudaMemcpyAsync(dst.p, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
}

void finish_disc(hdgb_ctx* c, hdgb_disc* d, int n_comp) {
    const HostMesh& m = d->mesh;
    const MasterElement& me = d->me;
    d->ctx = c;
    hdgb_dims& dm = d->dims;
    dm.dim = m.dim; dm.shape = m.shape; dm.degree = me.degree; dm.n_comp = n_comp;
    dm.ne = m.ne; dm.nf = m.nf; dm.n_lfe = m.n_lfe; dm.n_orient = me.n_orient;
    dm.pe = me.pe; dm.pf = me.pf; dm.qe = me.qe; dm.qf = me.qf; dm.nv = m.nv;

    d->geom = compute_geometry(m, me);
    DiscView& v = d->view;
    v.D = m.dim; v.M = n_comp; v.ne = m.ne; v.nf = m.nf; v.n_lfe = m.n_lfe; v.n_orient = me.n_orient;
    v.pe = me.pe; v.pf = me.pf; v.qe = me.qe; v.qf = me.qf;
    v.npe = n_comp * me.pe; v.mpf = n_comp * me.pf; v.nfl = m.n_lfe * v.mpf; v.nfs = m.n_lfe * me.pf;
    if (d->ne_owned < 0) d->ne_owned = m.ne;
    if (d->nf_owned < 0) d->nf_owned = m.nf;
    v.ne_owned = d->ne_owned;
    v.nf_owned = d->nf_owned;
    if (d->nf_global < 0) d->nf_global = m.nf;
    // Domain decomposition: the leading elements whose faces are all owned, and the leading owned faces whose block
    // row references owned faces only, need no halo data -- they run while the halo exchange is in flight
    // (partition.py numbers them first; a caller's own numbering just gets a shorter prefix, down to none).
    d->ne_interior = 0;
    d->nf_interior = 0;
    if (d->nf_owned < m.nf) {
        std::vector<char> elem_int(m.ne, 1);
        for (int e = 0; e < m.ne; ++e)
            for (int l = 0; l < m.n_lfe; ++l)
                if (m.elem_faces[static_cast<size_t>(e) * m.n_lfe + l] >= d->nf_owned) elem_int[e] = 0;
        while (d->ne_interior < d->ne_owned && elem_int[d->ne_interior]) ++d->ne_interior;
        auto face_int = [&](int f) {
            for (int s = 0; s < 2; ++s) {
                const int e = m.face_elems[2 * static_cast<size_t>(f) + s];
                if (e >= 0 && !elem_int[e]) return false;
            }
            return true;
        };
        while (d->nf_interior < d->nf_owned && face_int(d->nf_interior)) ++d->nf_interior;
    }
    if (!c) return;  // host-only discretisation: tables for inspection, no device state
    upload(c, d->elem_faces, m.elem_faces);
    upload(c, d->elem_side, m.elem_side);
    upload(c, d->face_elems, m.face_elems);
    upload(c, d->face_lidx, m.face_lidx);
    upload(c, d->face_orient, m.face_orient);
    upload(c, d->bnd_tag, m.bnd_tag);
    upload(c, d->phi, me.phi);
    for (int k = 0; k < m.dim; ++k) upload(c, d->dphi[k], me.dphi[k]);
    upload(c, d->psi, me.psi);
    upload(c, d->tphi, me.tphi);
    upload(c, d->wq, me.elem_wts);
    upload(c, d->wf, me.face_wts);
    upload(c, d->elem_detjac, d->geom.elem_detjac);
    upload(c, d->elem_invjac, d->geom.elem_invjac);
    upload(c, d->elem_coords, d->geom.elem_coords);
    upload(c, d->face_detjac, d->geom.face_detjac);
    upload(c, d->face_coords, d->geom.face_coords);
    upload(c, d->face_normal, d->geom.face_normal);

    v.elem_faces = d->elem_faces.p; v.elem_side = d->elem_side.p; v.face_elems = d->face_elems.p;
    v.face_lidx = d->face_lidx.p; v.face_orient = d->face_orient.p; v.bnd_tag = d->bnd_tag.p;
    v.phi = d->phi.p;
    for (int k = 0; k < 3; ++k) v.dphi[k] = d->dphi[k].p;
    v.psi = d->psi.p; v.tphi = d->tphi.p; v.wq = d->wq.p; v.wf = d->wf.p;
    v.es_vol = nullptr;
    v.es_face = nullptr;
    if (me.pe == 64) {
        // padded table images for the streamed E / D_d sweep of the local kernel (k_local.cu: ed_stream)
        constexpr int kPts = 8, kLd = 68;
        const int qe = static_cast<int>(me.elem_wts.size());
        const int nsv = (qe + kPts - 1) / kPts, nt = 1 + m.dim;
        std::vector<double> ev(static_cast<size_t>(nsv) * nt * kPts * kLd, 0.0);
        for (int s = 0; s < nsv; ++s)
            for (int k = 0; k < nt; ++k)
                for (int p = 0; p < kPts; ++p) {
                    const int g = std::min(s * kPts + p, qe - 1);
                    const std::vector<double>& tab = k == 0 ? me.phi : me.dphi[k - 1];
                    std::copy(tab.begin() + static_cast<size_t>(me.pe) * g, tab.begin() + static_cast<size_t>(me.pe) * (g + 1),
                              ev.begin() + ((static_cast<size_t>(s) * nt + k) * kPts + p) * kLd);
                }
        const size_t rows = me.tphi.size() / me.pe;
        std::vector<double> ef((rows + 8) * kLd, 0.0);  // + 8 zero rows: a face stage copies up to 4 ceil(qf / 4) rows
        for (size_t r = 0; r < rows; ++r)
            std::copy(me.tphi.begin() + r * me.pe, me.tphi.begin() + (r + 1) * me.pe, ef.begin() + r * kLd);
        upload(c, d->es_vol, ev);
        upload(c, d->es_face, ef);
        v.es_vol = d->es_vol.p;
        v.es_face = d->es_face.p;
    }
    v.elem_detjac = d->elem_detjac.p; v.elem_invjac = d->elem_invjac.p; v.elem_coords = d->elem_coords.p;
    v.face_detjac = d->face_detjac.p; v.face_coords = d->face_coords.p; v.face_normal = d->face_normal.p;

    // precompute_local_factors (local_ops.cpp:252-349) on the device.
    const size_t pp = static_cast<size_t>(me.pe) * me.pe * m.ne;
    const size_t pc = static_cast<size_t>(me.pe) * v.nfs * m.ne;
    d->mass.alloc(pp);
    d->mass_inv.alloc(pp);
    double* bm[3] = {nullptr, nullptr, nullptr};
    double* cm[3] = {nullptr, nullptr, nullptr};
    for (int k = 0; k < m.dim; ++k) {
        d->bmat[k].alloc(pp); d->cmat[k].alloc(pc); d->minv_b[k].alloc(pp); d->minv_c[k].alloc(pc);
        bm[k] = d->bmat[k].p; cm[k] = d->cmat[k].p;
    }
    launch_local_factors(c, v, d->mass.p, bm, cm);
    device_lu_invert(c, me.pe, m.ne, d->mass.p, d->mass_inv.p, "precompute_local_factors", HDGB_ERR_SINGULAR_MASS);
    for (int k = 0; k < m.dim; ++k) {
        launch_gemm_batch(c, me.pe, me.pe, me.pe, d->mass_inv.p, static_cast<int64_t>(me.pe) * me.pe, false,
                          d->bmat[k].p, static_cast<int64_t>(me.pe) * me.pe, d->minv_b[k].p,
                          static_cast<int64_t>(me.pe) * me.pe, m.ne, 1.0, 0.0);
        launch_gemm_batch(c, me.pe, v.nfs, me.pe, d->mass_inv.p, static_cast<int64_t>(me.pe) * me.pe, false,
                          d->cmat[k].p, static_cast<int64_t>(me.pe) * v.nfs, d->minv_c[k].p,
                          static_cast<int64_t>(me.pe) * v.nfs, m.ne, 1.0, 0.0);
        v.minv_b[k] = d->minv_b[k].p;
        v.minv_c[k] = d->minv_c[k].p;
    }
    HDGB_CUDA(cudaStreamSynchronize(c->stream));
}

template <class T>
hdgb_status get_vec(const hdgb_disc* d, const std::vector<T>& v, T* out, int64_t cap, int64_t* n) {
    if (n) *n = static_cast<int64_t>(v.size());
    if (out) {
        if (cap < static_cast<int64_t>(v.size())) {
            if (d->ctx) d->ctx->err = "destination too small";
            return HDGB_ERR_DIMENSION_MISMATCH;
        }
        std::memcpy(out, v.data(), v.size() * sizeof(T));
    }
    return HDGB_OK;
}

hdgb_status get_dev(const hdgb_disc* d, const DevBuf<double>& b, double* out, int64_t cap, int64_t* n) {
    if (!d->ctx) return HDGB_ERR_CUDA;  // device tables do not exist on a host-only discretisation
    if (n) *n = static_cast<int64_t>(b.n);
    if (out) {
        if (cap < static_cast<int64_t>(b.n)) {
            d->ctx->err = "destination too small";
            return HDGB_ERR_DIMENSION_MISMATCH;
        }
        return guarded(d->ctx, [&] {
            HDGB_CUDA(cudaMemcpyAsync(out, b.p, b.n * sizeof(double), cudaMemcpyDeviceToHost, d->ctx->stream));
            HDGB_CUDA(cudaStreamSynchronize(d->ctx->stream));
        });
    }
    return HDGB_OK;
}

}  // namespace

extern "C" {

hdgb_status hdgb_disc_create_structured(hdgb_ctx* c, int shape, int n, int degree, int n_comp, int quad_points,
                                        const double* lo, const double* hi, double jitter, uint64_t seed,
                                        hdgb_disc** out) {
    *out = nullptr;
    hdgb_disc* d = new hdgb_disc();
    hdgb_status st = guarded(c, [&] {
        if (n_comp < 1) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "n_comp must be >= 1");
        const double lo0[3] = {0, 0, 0}, hi0[3] = {1, 1, 1};
        d->me = make_master_element(shape, degree, quad_points);
        d->mesh = build_structured_mesh(shape, n, lo ? lo : lo0, hi ? hi : hi0, jitter, seed);
        finish_disc(c, d, n_comp);
    });
    if (st != HDGB_OK) { delete d; return st; }
    *out = d;
    return HDGB_OK;
}

hdgb_status hdgb_disc_create_from_mesh(hdgb_ctx* c, int shape, int degree, int n_comp, int quad_points, int ne,
                                       int nv, const int32_t* elem_verts, const double* vertex_coords,
                                       hdgb_disc** out) {
    *out = nullptr;
    hdgb_disc* d = new hdgb_disc();
    hdgb_status st = guarded(c, [&] {
        d->me = make_master_element(shape, degree, quad_points);
        d->mesh = build_mesh_from_elements(shape, ne, nv, elem_verts, vertex_coords);
        finish_disc(c, d, n_comp);
    });
    if (st != HDGB_OK) { delete d; return st; }
    *out = d;
    return HDGB_OK;
}

hdgb_status hdgb_disc_create_from_tables(hdgb_ctx* c, int shape, int degree, int n_comp, int quad_points, int ne, int nf,
                                         int nv, const int32_t* elem_verts, const double* vertex_coords,
                                         const int32_t* element_to_face, const int32_t* face_to_elements,
                                         const int32_t* face_local_index, const int32_t* face_orient,
                                         const int32_t* face_vertices, const int32_t* boundary_tag, int ne_owned,
                                         int nf_owned, const int64_t* face_gid, int64_t nf_global, hdgb_disc** out) {
    *out = nullptr;
    hdgb_disc* d = new hdgb_disc();
    hdgb_status st = guarded(c, [&] {
        if (ne_owned < 0 || ne_owned > ne || nf_owned < 0 || nf_owned > nf)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "dimension mismatch: owned element / face counts");
        d->me = make_master_element(shape, degree, quad_points);
        d->mesh = mesh_from_tables(shape, ne, nf, nv, elem_verts, vertex_coords, element_to_face, face_to_elements,
                                   face_local_index, face_orient, face_vertices, boundary_tag);
        d->ne_owned = ne_owned;
        d->nf_owned = nf_owned;
        if (face_gid) d->face_gid.assign(face_gid, face_gid + nf);
        d->nf_global = face_gid ? nf_global : nf;
        finish_disc(c, d, n_comp);
    });
    if (st != HDGB_OK) { delete d; return st; }
    *out = d;
    return HDGB_OK;
}

hdgb_status hdgb_mesh_connectivity(int shape, int ne, int nv, const int32_t* elem_verts, const double* vertex_coords,
                                   hdgb_disc** out) {
    *out = nullptr;
    hdgb_disc* d = new hdgb_disc();
    hdgb_status st = guarded(nullptr, [&] {
        d->mesh = build_mesh_from_elements(shape, ne, nv, elem_verts, vertex_coords);
        hdgb_dims& dm = d->dims;
        dm.dim = d->mesh.dim; dm.shape = shape; dm.ne = d->mesh.ne; dm.nf = d->mesh.nf; dm.n_lfe = d->mesh.n_lfe; dm.nv = nv;
        dm.n_comp = 1;
    });
    if (st != HDGB_OK) { delete d; return st; }
    *out = d;
    return HDGB_OK;
}

void hdgb_disc_destroy(hdgb_disc* d) { delete d; }

hdgb_status hdgb_disc_dims(const hdgb_disc* d, hdgb_dims* out) {
    *out = d->dims;
    return HDGB_OK;
}

hdgb_status hdgb_disc_set_boundary_tags(hdgb_disc* d, const int32_t* tags) {
    return guarded(d->ctx, [&] {
        for (int f = 0; f < d->mesh.nf; ++f)
            if (d->mesh.face_elems[2 * f + 1] < 0) d->mesh.bnd_tag[f] = tags[f];
        upload(d->ctx, d->bnd_tag, d->mesh.bnd_tag);
        d->view.bnd_tag = d->bnd_tag.p;
        HDGB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    });
}

hdgb_status hdgb_disc_get_i32(const hdgb_disc* d, const char* name, int32_t* out, int64_t cap, int64_t* n) {
    const std::string s = name;
    const HostMesh& m = d->mesh;
    if (s == "interior_counts") return get_vec(d, std::vector<int>{d->ne_interior, d->nf_interior}, out, cap, n);
    if (s == "element_to_face") return get_vec(d, m.elem_faces, out, cap, n);
    if (s == "element_vertices") return get_vec(d, m.elem_verts, out, cap, n);
    if (s == "face_to_elements") return get_vec(d, m.face_elems, out, cap, n);
    if (s == "face_local_index") return get_vec(d, m.face_lidx, out, cap, n);
    if (s == "face_orient") return get_vec(d, m.face_orient, out, cap, n);
    if (s == "face_vertices") return get_vec(d, m.face_verts, out, cap, n);
    if (s == "boundary_tag") return get_vec(d, m.bnd_tag, out, cap, n);
    if (s == "elem_side") return get_vec(d, m.elem_side, out, cap, n);
    if (s == "qperm") return get_vec(d, d->me.qperm, out, cap, n);
    if (d->ctx) d->ctx->err = "unknown int table '" + s + "'";
    return HDGB_ERR_GENERIC;
}

hdgb_status hdgb_disc_get_f64(const hdgb_disc* d, const char* name, double* out, int64_t cap, int64_t* n) {
    const std::string s = name;
    const MasterElement& me = d->me;
    const HostGeom& g = d->geom;
    if (s == "phi") return get_vec(d, me.phi, out, cap, n);
    if (s == "dphi0") return get_vec(d, me.dphi[0], out, cap, n);
    if (s == "dphi1") return get_vec(d, me.dphi[1], out, cap, n);
    if (s == "dphi2") return get_vec(d, me.dphi[2], out, cap, n);
    if (s == "psi") return get_vec(d, me.psi, out, cap, n);
    if (s == "tphi") return get_vec(d, me.tphi, out, cap, n);
    if (s == "tphi_local") return get_vec(d, me.tphi_local, out, cap, n);
    if (s == "nodes1d") return get_vec(d, me.nodes1d, out, cap, n);
    if (s == "elem_nodes") return get_vec(d, me.elem_nodes, out, cap, n);
    if (s == "face_nodes") return get_vec(d, me.face_nodes, out, cap, n);
    if (s == "rule1d_points") return get_vec(d, me.rule1d.pts, out, cap, n);
    if (s == "rule1d_weights") return get_vec(d, me.rule1d.wts, out, cap, n);
    if (s == "elem_points") return get_vec(d, me.elem_pts, out, cap, n);
    if (s == "elem_weights") return get_vec(d, me.elem_wts, out, cap, n);
    if (s == "face_points") return get_vec(d, me.face_pts, out, cap, n);
    if (s == "face_weights") return get_vec(d, me.face_wts, out, cap, n);
    if (s == "vertex_coords") return get_vec(d, d->mesh.coords, out, cap, n);
    if (s == "elem_detjac") return get_vec(d, g.elem_detjac, out, cap, n);
    if (s == "elem_invjac") return get_vec(d, g.elem_invjac, out, cap, n);
    if (s == "elem_coords") return get_vec(d, g.elem_coords, out, cap, n);
    if (s == "face_detjac") return get_vec(d, g.face_detjac, out, cap, n);
    if (s == "face_coords") return get_vec(d, g.face_coords, out, cap, n);
    if (s == "face_normal") return get_vec(d, g.face_normal, out, cap, n);
    if (s == "mass") return get_dev(d, d->mass, out, cap, n);
    if (s == "mass_inv") return get_dev(d, d->mass_inv, out, cap, n);
    for (int k = 0; k < 3; ++k) {
        const std::string ks = std::to_string(k);
        if (s == "bmat" + ks) return get_dev(d, d->bmat[k], out, cap, n);
        if (s == "cmat" + ks) return get_dev(d, d->cmat[k], out, cap, n);
        if (s == "minv_b" + ks) return get_dev(d, d->minv_b[k], out, cap, n);
        if (s == "minv_c" + ks) return get_dev(d, d->minv_c[k], out, cap, n);
    }
    if (d->ctx) d->ctx->err = "unknown table '" + s + "'";
    return HDGB_ERR_GENERIC;
}

// ---- model ------------------------------------------------------------------------------------------
hdgb_status hdgb_model_create(hdgb_ctx* c, const hdgb_disc* d, int kind, const double* params, int n_params,
                              const double* forcing_q, const double* dirichlet_q, hdgb_model** out) {
    *out = nullptr;
    hdgb_model* m = new hdgb_model();
    hdgb_status st = guarded(c, [&] {
        m->ctx = c;
        m->view.kind = kind;
        for (int i = 0; i < 16; ++i) m->view.p[i] = (params && i < n_params) ? params[i] : 0.0;
        const int M = d->dims.n_comp;
        const int need = (kind == HDGB_MODEL_ELASTICITY) ? d->dims.dim : (kind == HDGB_MODEL_NAVIER_STOKES ? d->dims.dim + 2 : 1);
        if (M != need)
            throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "model needs " + std::to_string(need) +
                                                           " components, discretisation has " + std::to_string(M));
        if (kind < 0 || kind > HDGB_MODEL_NAVIER_STOKES) throw Failure(HDGB_ERR_UNSUPPORTED, "unknown model kind");
        m->n_comp = M;
        if (forcing_q) {
            m->forcing_q.alloc(static_cast<size_t>(d->dims.ne) * d->dims.qe * M);
            m->forcing_q.upload(forcing_q, m->forcing_q.n, c->stream);
        }
        if (dirichlet_q) {
            m->dirichlet_q.alloc(static_cast<size_t>(d->dims.nf) * d->dims.qf * M);
            m->dirichlet_q.upload(dirichlet_q, m->dirichlet_q.n, c->stream);
        }
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        m->view.forcing_q = m->forcing_q.p;
        m->view.dirichlet_q = m->dirichlet_q.p;
    });
    if (st != HDGB_OK) { delete m; return st; }
    *out = m;
    return HDGB_OK;
}

void hdgb_model_destroy(hdgb_model* m) { delete m; }

// ---- state ------------------------------------------------------------------------------------------
hdgb_status hdgb_state_create(hdgb_ctx* c, const hdgb_disc* d, hdgb_state** out) {
    *out = nullptr;
    hdgb_state* s = new hdgb_state();
    hdgb_status st = guarded(c, [&] {
        s->ctx = c;
        s->disc = d;
        const size_t nu = static_cast<size_t>(d->view.npe) * d->dims.ne;
        s->u.alloc(nu);
        s->u.zero(c->stream);
        for (int k = 0; k < d->dims.dim; ++k) { s->q[k].alloc(nu); s->q[k].zero(c->stream); }
        s->uhat.alloc(static_cast<size_t>(d->view.mpf) * d->dims.nf);
        s->uhat.zero(c->stream);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
    if (st != HDGB_OK) { delete s; return st; }
    *out = s;
    return HDGB_OK;
}

void hdgb_state_destroy(hdgb_state* s) { delete s; }

static DevBuf<double>* state_field(hdgb_state* s, const char* name) {
    const std::string n = name;
    if (n == "u") return &s->u;
    if (n == "uhat") return &s->uhat;
    if (n == "q0") return &s->q[0];
    if (n == "q1") return &s->q[1];
    if (n == "q2") return &s->q[2];
    return nullptr;
}

hdgb_status hdgb_state_set(hdgb_state* s, const char* name, const double* src) {
    return guarded(s->ctx, [&] {
        DevBuf<double>* b = state_field(s, name);
        if (!b || !b->p) throw Failure(HDGB_ERR_GENERIC, std::string("unknown state field ") + name);
        HDGB_CUDA(cudaMemcpyAsync(b->p, src, b->n * sizeof(double), cudaMemcpyDefault, s->ctx->stream));
        HDGB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    });
}

hdgb_status hdgb_state_get(const hdgb_state* s, const char* name, double* dst) {
    return guarded(s->ctx, [&] {
        DevBuf<double>* b = state_field(const_cast<hdgb_state*>(s), name);
        if (!b || !b->p) throw Failure(HDGB_ERR_GENERIC, std::string("unknown state field ") + name);
        HDGB_CUDA(cudaMemcpyAsync(dst, b->p, b->n * sizeof(double), cudaMemcpyDefault, s->ctx->stream));
        HDGB_CUDA(cudaStreamSynchronize(s->ctx->stream));
    });
}

double* hdgb_state_ptr(hdgb_state* s, const char* name) {
    DevBuf<double>* b = state_field(s, name);
    return b ? b->p : nullptr;
}

}  // extern "C"

// ---- local operators -----------------------------------------------------------------------------------
namespace hdgb {

void compute_q_device(hdgb_disc* d, hdgb_state* s) {
    hdgb_ctx* c = d->ctx;
    const DiscView& v = d->view;
    const int64_t batch = static_cast<int64_t>(v.ne) * v.M;
    for (int k = 0; k < v.D; ++k) {
        GemvArgs g;
        g.a = v.minv_b[k]; g.x = s->u.p; g.y = s->q[k].p;
        g.rows = v.pe; g.cols = v.pe; g.batch = batch; g.a_div = v.M;
        g.alpha = -1.0;
        launch_team_gemv(c, g);
        GemvArgs h;
        h.a = v.minv_c[k]; h.x = s->uhat.p; h.y = s->q[k].p; h.z = s->q[k].p;
        h.rows = v.pe; h.cols = v.nfs; h.batch = batch; h.a_div = v.M;
        h.idx = v.elem_faces; h.width = v.pf; h.comp = v.M;
        h.alpha = -1.0; h.beta = 1.0;
        launch_team_gemv(c, h);
    }
}

void check_state_finite(hdgb_disc* d, hdgb_state* s) {
    hdgb_ctx* c = d->ctx;
    // local_ops.cpp:36-37 checks u first, then uhat
    reset_flags(c);
    launch_check_finite(c, s->u.p, static_cast<int64_t>(s->u.n), c->d_flags);
    int bad = 0;
    read_flags(c, nullptr, &bad);
    if (bad) throw Failure(HDGB_ERR_NONFINITE_STATE, "non-finite state: interior solution");
    reset_flags(c);
    launch_check_finite(c, s->uhat.p, static_cast<int64_t>(s->uhat.n), c->d_flags);
    read_flags(c, nullptr, &bad);
    if (bad) throw Failure(HDGB_ERR_NONFINITE_STATE, "non-finite state: trace solution");
}

// Runs assemble_core for elements [e0, e0+cnt) (raw blocks chunk-local, residual vectors global).
static void run_assemble(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, const double* u_prev, double dt_inv,
                         int e0, int cnt, const LocalOut& out, bool want_jac) {
    DiscView v = d->view;
    // shift the element-indexed tables so that blockIdx.x == 0 addresses element e0
    v.ne = cnt;
    v.elem_faces += static_cast<size_t>(e0) * v.n_lfe;
    v.elem_side += static_cast<size_t>(e0) * v.n_lfe;
    v.elem_detjac += static_cast<size_t>(e0) * v.qe;
    v.elem_invjac += static_cast<size_t>(e0) * v.qe * v.D * v.D;
    v.elem_coords += static_cast<size_t>(e0) * v.qe * v.D;
    ModelView mv = m->view;
    if (mv.forcing_q) mv.forcing_q += static_cast<size_t>(e0) * v.qe * v.M;
    LocalIn in{};
    in.u = s->u.p + static_cast<size_t>(e0) * v.npe;
    for (int k = 0; k < v.D; ++k) in.q[k] = s->q[k].p + static_cast<size_t>(e0) * v.npe;
    in.uhat = s->uhat.p;
    in.u_prev = u_prev ? u_prev + static_cast<size_t>(e0) * v.npe : nullptr;
    in.dt_inv = dt_inv;
    LocalOut o = out;
    o.ru += static_cast<size_t>(e0) * v.npe;
    o.ruhat_e += static_cast<size_t>(e0) * v.nfl;
    launch_local_assemble(d->ctx, v, mv, in, o, want_jac);
}


double assemble_residual_device(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, const double* u_prev_dev,
                                double dt, double* trace, double* interior) {
    hdgb_ctx* c = d->ctx;
    const DiscView& v = d->view;
    check_state_finite(d, s);
    const bool transient = dt > 0.0;
    if (transient && !u_prev_dev)
        throw Failure(HDGB_ERR_INCONSISTENT_DIMENSIONS, "inconsistent dimensions: transient assembly requires the previous solution");
    compute_q_device(d, s);
    const size_t n_int = static_cast<size_t>(v.npe) * v.ne, n_tr = static_cast<size_t>(v.mpf) * v.nf;
    if (d->res_ruhat_e.n != static_cast<size_t>(v.nfl) * v.ne) {
        d->res_ruhat_e.alloc(static_cast<size_t>(v.nfl) * v.ne);
        d->res_partial.alloc(multi_dot_workspace_doubles(static_cast<int64_t>(std::max(n_int, n_tr)), 1));
        d->res_sums.alloc(2);
    }
    LocalOut lo{};
    lo.ru = interior;
    lo.ruhat_e = d->res_ruhat_e.p;
    run_assemble(d, m, s, u_prev_dev, transient ? 1.0 / dt : 0.0, 0, v.ne, lo, false);
    // face assembly of the trace residual (local_ops.cpp:439-447), side 0 then side 1; owned faces
    // have both sides local (the ghost layer is assembled redundantly)
    launch_face_sum(c, d->res_ruhat_e.p, v.face_elems, v.face_lidx, v.nf_owned, v.mpf, v.n_lfe, trace);
    // residual_norm (local_ops.cpp:245-250) over owned faces / elements (+ all-reduce across ranks)
    launch_sumsq(c, trace, static_cast<int64_t>(v.mpf) * v.nf_owned, d->res_sums.p, d->res_partial.p);
    launch_sumsq(c, interior, static_cast<int64_t>(v.npe) * v.ne_owned, d->res_sums.p + 1, d->res_partial.p);
    if (c->comm) c->comm->allreduce(c, d->res_sums.p, 2);
    double h[2];
    HDGB_CUDA(cudaMemcpyAsync(h, d->res_sums.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    HDGB_CUDA(cudaStreamSynchronize(c->stream));
    return std::sqrt(h[0] + h[1]);
}

void recover_local_device(hdgb_disc* d, const hdgb_ops* o, const double* duhat, double* du, double* tmp) {
    hdgb_ctx* c = d->ctx;
    const DiscView& v = d->view;
    // tmp = r_u - F-bar duhat_e  (gather fused), du = E-bar^-1 tmp   (local_ops.cpp:452-460)
    GemvArgs g1;
    g1.a = o->fbar.p; g1.x = duhat; g1.y = tmp; g1.z = o->ru.p;
    g1.rows = v.npe; g1.cols = v.nfl; g1.batch = v.ne;
    g1.idx = v.elem_faces; g1.width = v.mpf; g1.comp = 1;
    g1.alpha = -1.0; g1.beta = 1.0;
    launch_team_gemv(c, g1);
    GemvArgs g2;
    g2.a = o->ebar_inv.p; g2.x = tmp; g2.y = du;
    g2.rows = v.npe; g2.cols = v.npe; g2.batch = v.ne;
    launch_team_gemv(c, g2);
}

}  // namespace hdgb

extern "C" {

hdgb_status hdgb_compute_q(hdgb_disc* d, hdgb_state* s) {
    return guarded(d->ctx, [&] {
        compute_q_device(d, s);
        HDGB_CUDA(cudaStreamSynchronize(d->ctx->stream));
    });
}

}  // extern "C"

namespace hdgb {

hdgb_ops* assemble_element_operators_device(hdgb_disc* d, const hdgb_model* m, hdgb_state* s,
                                            const double* u_prev_dev, double dt, bool keep_raw) {
    hdgb_ctx* c = d->ctx;
    std::unique_ptr<hdgb_ops> holder(new hdgb_ops());
    hdgb_ops* o = holder.get();
    const DiscView& v = d->view;
    const int ne = v.ne, npe = v.npe, nfl = v.nfl, D = v.D, M = v.M, pe = v.pe, pf = v.pf, mpf = v.mpf;
    check_state_finite(d, s);
    const bool transient = dt > 0.0;
    if (transient && !u_prev_dev)
        throw Failure(HDGB_ERR_INCONSISTENT_DIMENSIONS, "inconsistent dimensions: transient assembly requires the previous solution");
    const double dt_inv = transient ? 1.0 / dt : 0.0;
    compute_q_device(d, s);

    o->ctx = c; o->npe = npe; o->nfl = nfl; o->ne = ne; o->D = D;
    const size_t sEE = static_cast<size_t>(npe) * npe, sEF = static_cast<size_t>(npe) * nfl, sFF = static_cast<size_t>(nfl) * nfl;
    o->kbar.alloc(sFF * ne);
    o->ebar_inv.alloc(sEE * ne);
    o->fbar.alloc(sEF * ne);
    o->hbar.alloc(sEF * ne);
    o->rbar.alloc(static_cast<size_t>(nfl) * ne);
    o->ru.alloc(static_cast<size_t>(npe) * ne);
    o->ruhat_e.alloc(static_cast<size_t>(nfl) * ne);

    // Raw-block workspace: bounded chunk of elements (whole mesh when the raw blocks are kept).
    const size_t per_elem = sEE * (1 + D) + sEF * (2 + D) + sFF;
    // the workspace may take up to a third of the free HBM (180 GB parts: config 2 runs in one chunk)
    // parked blocks of the caching allocator count as free: the chunking must not depend on what earlier calls left
    // cached, or buffer sizes change from call to call and every allocation misses the cache.  The budget is fixed
    // at the first assembly on this discretisation: cudaMemGetInfo is a resource-manager call that queues behind
    // any concurrent nvidia-smi / NVML query on the box (measured: sporadic +15..55 ms per Newton iteration while a
    // monitor polls the GPU), so it stays out of the steady-state path.
    if (d->assemble_budget <= 0.0) {
        size_t free_b = 0, total_b = 0;
        HDGB_CUDA(cudaMemGetInfo(&free_b, &total_b));
        d->assemble_budget = std::max(2.0e9, static_cast<double>(free_b + pool_parked_bytes()) / 3.0);
    }
    const double budget = d->assemble_budget;
    size_t chunk = keep_raw ? ne : static_cast<size_t>(budget / (per_elem * sizeof(double)));
    if (chunk < 1) chunk = 1;
    if (chunk > static_cast<size_t>(ne)) chunk = ne;
    DevBuf<double> wE, wD[3], wG[3], wJ, wT;
    DevBuf<double>*pE = &wE, *pJ = &wJ;
    DevBuf<double>* pD[3] = {&wD[0], &wD[1], &wD[2]};
    DevBuf<double>* pG[3] = {&wG[0], &wG[1], &wG[2]};
    if (keep_raw) {
        o->has_raw = true;
        o->e_raw.alloc(sEE * ne); o->f_raw.alloc(sEF * ne); o->h_raw.alloc(sEF * ne); o->j_raw.alloc(sFF * ne);
        for (int k = 0; k < D; ++k) { o->d_raw[k].alloc(sEE * ne); o->g_raw[k].alloc(sEF * ne); }
        pD[0] = &o->d_raw[0]; pD[1] = &o->d_raw[1]; pD[2] = &o->d_raw[2];
        pG[0] = &o->g_raw[0]; pG[1] = &o->g_raw[1]; pG[2] = &o->g_raw[2];
    } else {
        for (int k = 0; k < D; ++k) { wD[k].alloc(sEE * chunk); wG[k].alloc(sEF * chunk); }
    }
    wE.alloc(sEE * chunk);  // becomes E-bar
    wJ.alloc(sFF * chunk);  // becomes J-bar, then K-bar is written to o->kbar
    wT.alloc(sEF * chunk);  // E-bar^-1 F-bar
    DevBuf<double> einv_ru(static_cast<size_t>(npe) * chunk);

    for (int e0 = 0; e0 < ne; e0 += static_cast<int>(chunk)) {
        const int cnt = static_cast<int>(std::min<size_t>(chunk, ne - e0));
        LocalOut lo{};
        lo.ru = o->ru.p;
        lo.ruhat_e = o->ruhat_e.p;
        lo.E = pE->p;
        lo.J = pJ->p;
        // F-bar and H-bar are assembled straight into their final storage
        lo.F = o->fbar.p + sEF * e0;
        lo.H = o->hbar.p + sEF * e0;
        for (int k = 0; k < D; ++k) {
            lo.Dm[k] = pD[k]->p + (keep_raw ? sEE * e0 : 0);
            lo.G[k] = pG[k]->p + (keep_raw ? sEF * e0 : 0);
        }
        run_assemble(d, m, s, u_prev_dev, dt_inv, e0, cnt, lo, true);
        if (keep_raw) {
            const size_t b = sizeof(double);
            HDGB_CUDA(cudaMemcpyAsync(o->e_raw.p + sEE * e0, lo.E, sEE * cnt * b, cudaMemcpyDeviceToDevice, c->stream));
            HDGB_CUDA(cudaMemcpyAsync(o->j_raw.p + sFF * e0, lo.J, sFF * cnt * b, cudaMemcpyDeviceToDevice, c->stream));
            HDGB_CUDA(cudaMemcpyAsync(o->f_raw.p + sEF * e0, lo.F, sEF * cnt * b, cudaMemcpyDeviceToDevice, c->stream));
            HDGB_CUDA(cudaMemcpyAsync(o->h_raw.p + sEF * e0, lo.H, sEF * cnt * b, cudaMemcpyDeviceToDevice, c->stream));
        }
        // q-elimination (local_ops.cpp:389-398): X-bar = X - sum_d Y_d (I_M (x) M^-1 B_d | M^-1 C_d)
        const int64_t sb = static_cast<int64_t>(pe) * pe, sc = static_cast<int64_t>(pe) * v.nfs;
        bool fused = false;
        if (tuning().use_dmma && tuning().use_qelim_fused && (tuning().qelim_split_rows || (npe + 31) / 32 + (nfl + 31) / 32 <= 8)) {
            // two stacked products per component column block: [E-bar; H-bar] -= sum_d [D_d; G_d] M^-1 B_d and
            // [F-bar; J-bar] -= sum_d [D_d; G_d] M^-1 C_d, the latter scattering its columns (lf, b) to
            // lf*mpf + mp*pf + b
            fused = true;
            for (int mp = 0; mp < M && fused; ++mp) {
                const size_t colblk = static_cast<size_t>(mp) * pe;
                const double *a0[3] = {nullptr, nullptr, nullptr}, *a1[3] = {nullptr, nullptr, nullptr};
                const double *bb[3] = {nullptr, nullptr, nullptr}, *bc[3] = {nullptr, nullptr, nullptr};
                for (int k = 0; k < D; ++k) {
                    a0[k] = lo.Dm[k] + colblk * npe;
                    a1[k] = lo.G[k] + colblk * nfl;
                    bb[k] = v.minv_b[k] + sb * e0;
                    bc[k] = v.minv_c[k] + sc * e0;
                }
                if (tuning().qelim_split_rows) {
                    // one product per output block, all D directions in its K sweep: smaller CTAs, more of them per SM
                    fused = launch_qelim_fused(c, npe, 0, pe, pe, D, a0, sEE, a0, sEE, bb, sb, lo.E + colblk * npe, sEE, nullptr, 0, cnt) &&
                            launch_qelim_fused(c, nfl, 0, pe, pe, D, a1, sEF, a1, sEF, bb, sb, lo.H + colblk * nfl, sEF, nullptr, 0, cnt) &&
                            launch_qelim_fused(c, npe, 0, v.nfs, pe, D, a0, sEE, a0, sEE, bc, sc,
                                               lo.F + static_cast<size_t>(mp) * pf * npe, sEF, nullptr, 0, cnt, pf, mpf) &&
                            launch_qelim_fused(c, nfl, 0, v.nfs, pe, D, a1, sEF, a1, sEF, bc, sc,
                                               lo.J + static_cast<size_t>(mp) * pf * nfl, sFF, nullptr, 0, cnt, pf, mpf);
                    continue;
                }
                fused = launch_qelim_fused(c, npe, nfl, pe, pe, D, a0, sEE, a1, sEF, bb, sb, lo.E + colblk * npe, sEE,
                                           lo.H + colblk * nfl, sEF, cnt);
                if (fused)
                    launch_qelim_fused(c, npe, nfl, v.nfs, pe, D, a0, sEE, a1, sEF, bc, sc, lo.F + static_cast<size_t>(mp) * pf * npe,
                                       sEF, lo.J + static_cast<size_t>(mp) * pf * nfl, sFF, cnt, pf, mpf);
            }
        }
        for (int k = 0; k < D && !fused; ++k) {
            const double* mb = v.minv_b[k] + sb * e0;
            const double* mc = v.minv_c[k] + sc * e0;
            for (int mp = 0; mp < M; ++mp) {
                const size_t colblk = static_cast<size_t>(mp) * pe;
                // E-bar[:, mp block] -= D_k[:, mp block] * minv_b
                launch_gemm_batch(c, npe, pe, pe, lo.Dm[k] + colblk * npe, sEE, false, mb, sb,
                                  lo.E + colblk * npe, sEE, cnt, -1.0, 1.0);
                // H-bar[:, mp block] -= G_k[:, mp block] * minv_b
                launch_gemm_batch(c, nfl, pe, pe, lo.G[k] + colblk * nfl, sEF, false, mb, sb,
                                  lo.H + colblk * nfl, sEF, cnt, -1.0, 1.0);
                if (M == 1) {
                    launch_gemm_batch(c, npe, nfl, pe, lo.Dm[k], sEE, false, mc, sc, lo.F, sEF, cnt, -1.0, 1.0);
                    launch_gemm_batch(c, nfl, nfl, pe, lo.G[k], sEF, false, mc, sc, lo.J, sFF, cnt, -1.0, 1.0);
                } else if (tuning().use_dmma) {
                    // all local faces in one product: B = M^-1 C_d (pe x n_lfe pf); output column (lf, b)
                    // lands in column lf*mpf + mp*pf + b of F-bar / J-bar
                    launch_gemm_dmma(c, npe, v.nfs, pe, lo.Dm[k] + colblk * npe, sEE, mc, sc,
                                     lo.F + static_cast<size_t>(mp) * pf * npe, sEF, cnt, -1.0, 1.0, pf, mpf);
                    launch_gemm_dmma(c, nfl, v.nfs, pe, lo.G[k] + colblk * nfl, sEF, mc, sc,
                                     lo.J + static_cast<size_t>(mp) * pf * nfl, sFF, cnt, -1.0, 1.0, pf, mpf);
                } else {
                    for (int lf = 0; lf < v.n_lfe; ++lf) {
                        const size_t tcol = static_cast<size_t>(lf) * mpf + static_cast<size_t>(mp) * pf;
                        launch_gemm_batch(c, npe, pf, pe, lo.Dm[k] + colblk * npe, sEE, false,
                                          mc + static_cast<size_t>(lf) * pf * pe, sc, lo.F + tcol * npe, sEF, cnt, -1.0, 1.0);
                        launch_gemm_batch(c, nfl, pf, pe, lo.G[k] + colblk * nfl, sEF, false,
                                          mc + static_cast<size_t>(lf) * pf * pe, sc, lo.J + tcol * nfl, sFF, cnt, -1.0, 1.0);
                    }
                }
            }
        }
        // E-bar^-1 (local_ops.cpp:400-404)
        reset_flags(c);
        launch_lu_invert_batch(c, npe, cnt, lo.E, o->ebar_inv.p + sEE * e0, c->d_flags);
        int bad = -1;
        read_flags(c, &bad, nullptr);
        if (bad >= 0)
            throw Failure(HDGB_ERR_SINGULAR_LOCAL_SOLVE, "singular local solve in element " + std::to_string(e0 + bad), e0 + bad);
        // K-bar = J-bar - H-bar (E-bar^-1 F-bar)   (local_ops.cpp:408-411)
        const bool schur_dmma = tuning().use_dmma && nfl * nfl > 256;
        if (schur_dmma && tuning().schur_fused &&
            launch_schur_fused(c, npe, nfl, o->ebar_inv.p + sEE * e0, sEE, lo.F, lo.H, sEF, lo.J, o->kbar.p + sFF * e0, sFF, cnt)) {
            // one kernel: T = E-bar^-1 F-bar stays in shared memory, J-bar is read in the epilogue
        } else {
            launch_gemm_batch(c, npe, nfl, npe, o->ebar_inv.p + sEE * e0, sEE, false, lo.F, sEF, wT.p, sEF, cnt, 1.0, 0.0);
            if (schur_dmma) {
                // K-bar = 1 * J-bar - H-bar T: the J-bar term is read in the epilogue, no copy of J-bar into K-bar first
                launch_gemm_dmma(c, nfl, nfl, npe, lo.H, sEF, wT.p, sEF, o->kbar.p + sFF * e0, sFF, cnt, -1.0, 1.0, 0, 0, lo.J);
            } else {
                HDGB_CUDA(cudaMemcpyAsync(o->kbar.p + sFF * e0, lo.J, sFF * cnt * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
                launch_gemm_batch(c, nfl, nfl, npe, lo.H, sEF, false, wT.p, sEF, o->kbar.p + sFF * e0, sFF, cnt, -1.0, 1.0);
            }
        }
        // r-bar = r_uhat - H-bar (E-bar^-1 r_u)   (local_ops.cpp:413-418)
        GemvArgs g1;
        g1.a = o->ebar_inv.p + sEE * e0; g1.x = o->ru.p + static_cast<size_t>(npe) * e0; g1.y = einv_ru.p;
        g1.rows = npe; g1.cols = npe; g1.batch = cnt;
        launch_team_gemv(c, g1);
        GemvArgs g2;
        g2.a = lo.H; g2.x = einv_ru.p; g2.y = o->rbar.p + static_cast<size_t>(nfl) * e0;
        g2.z = o->ruhat_e.p + static_cast<size_t>(nfl) * e0;
        g2.rows = nfl; g2.cols = npe; g2.batch = cnt; g2.alpha = -1.0; g2.beta = 1.0;
        launch_team_gemv(c, g2);
    }
    return holder.release();
}

}  // namespace hdgb

extern "C" {

hdgb_status hdgb_assemble_element_operators(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, const hdgb_time* t,
                                            int keep_raw, hdgb_ops** out) {
    *out = nullptr;
    hdgb_ctx* c = d->ctx;
    return guarded(c, [&] {
        const bool transient = t && t->dt > 0.0;
        if (transient && !t->u_prev)
            throw Failure(HDGB_ERR_INCONSISTENT_DIMENSIONS, "inconsistent dimensions: transient assembly requires the previous solution");
        InArg uprev(c, transient ? t->u_prev : nullptr, static_cast<size_t>(d->view.npe) * d->view.ne);
        hdgb_ops* o = assemble_element_operators_device(d, m, s, uprev.dev, transient ? t->dt : 0.0, keep_raw != 0);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        *out = o;
    });
}

hdgb_status hdgb_ops_create(hdgb_disc* d, const double* kbar, const double* ebar_inv, const double* fbar, const double* hbar,
                            const double* rbar, const double* ru, const double* ruhat_e, hdgb_ops** out) {
    *out = nullptr;
    hdgb_ctx* c = d->ctx;
    return guarded(c, [&] {
        const DiscView& v = d->view;
        std::unique_ptr<hdgb_ops> o(new hdgb_ops());
        o->ctx = c; o->npe = v.npe; o->nfl = v.nfl; o->ne = v.ne; o->D = v.D;
        const size_t ne = v.ne, npe = v.npe, nfl = v.nfl;
        auto fill = [&](DevBuf<double>& b, const double* src, size_t n) {
            b.alloc(n);
            if (src) HDGB_CUDA(cudaMemcpyAsync(b.p, src, n * sizeof(double), cudaMemcpyDefault, c->stream));
            else b.zero(c->stream);
        };
        fill(o->kbar, kbar, nfl * nfl * ne);
        fill(o->ebar_inv, ebar_inv, npe * npe * ne);
        fill(o->fbar, fbar, npe * nfl * ne);
        fill(o->hbar, hbar, nfl * npe * ne);
        fill(o->rbar, rbar, nfl * ne);
        fill(o->ru, ru, npe * ne);
        fill(o->ruhat_e, ruhat_e, nfl * ne);
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
        *out = o.release();
    });
}

void hdgb_ops_destroy(hdgb_ops* o) { delete o; }

static hdgb::DevBuf<double>* ops_field(hdgb_ops* o, const char* name) {
    const std::string n = name;
    if (n == "kbar") return &o->kbar;
    if (n == "ebar_inv") return &o->ebar_inv;
    if (n == "fbar") return &o->fbar;
    if (n == "hbar") return &o->hbar;
    if (n == "rbar") return &o->rbar;
    if (n == "ru") return &o->ru;
    if (n == "ruhat_e") return &o->ruhat_e;
    if (n == "e_raw") return &o->e_raw;
    if (n == "f_raw") return &o->f_raw;
    if (n == "h_raw") return &o->h_raw;
    if (n == "j_raw") return &o->j_raw;
    for (int k = 0; k < 3; ++k) {
        if (n == "d_raw" + std::to_string(k)) return &o->d_raw[k];
        if (n == "g_raw" + std::to_string(k)) return &o->g_raw[k];
    }
    return nullptr;
}

hdgb_status hdgb_ops_get(const hdgb_ops* o, const char* name, double* dst, int64_t cap, int64_t* n) {
    return guarded(o->ctx, [&] {
        DevBuf<double>* b = ops_field(const_cast<hdgb_ops*>(o), name);
        if (!b) throw Failure(HDGB_ERR_GENERIC, std::string("unknown operator field ") + name);
        if (n) *n = static_cast<int64_t>(b->n);
        if (dst) {
            if (cap < static_cast<int64_t>(b->n)) throw Failure(HDGB_ERR_DIMENSION_MISMATCH, "destination too small");
            HDGB_CUDA(cudaMemcpyAsync(dst, b->p, b->n * sizeof(double), cudaMemcpyDeviceToHost, o->ctx->stream));
            HDGB_CUDA(cudaStreamSynchronize(o->ctx->stream));
        }
    });
}

double* hdgb_ops_ptr(hdgb_ops* o, const char* name) {
    DevBuf<double>* b = ops_field(o, name);
    return b ? b->p : nullptr;
}

hdgb_status hdgb_assemble_residual(hdgb_disc* d, const hdgb_model* m, hdgb_state* s, const hdgb_time* t,
                                   double* trace, double* interior, double* norm) {
    hdgb_ctx* c = d->ctx;
    return guarded(c, [&] {
        const DiscView& v = d->view;
        const bool transient = t && t->dt > 0.0;
        if (transient && !t->u_prev)
            throw Failure(HDGB_ERR_INCONSISTENT_DIMENSIONS, "inconsistent dimensions: transient assembly requires the previous solution");
        InArg uprev(c, transient ? t->u_prev : nullptr, static_cast<size_t>(v.npe) * v.ne);
        const size_t n_int = static_cast<size_t>(v.npe) * v.ne, n_tr = static_cast<size_t>(v.mpf) * v.nf;
        DevBuf<double> tr_tmp, in_tmp;
        OutArg T(c, trace, n_tr), I(c, interior, n_int);
        if (!T.dev) { tr_tmp.alloc(n_tr); T.dev = tr_tmp.p; }
        if (!I.dev) { in_tmp.alloc(n_int); I.dev = in_tmp.p; }
        const double nrm = assemble_residual_device(d, m, s, uprev.dev, transient ? t->dt : 0.0, T.dev, I.dev);
        if (norm) *norm = nrm;
        T.commit();
        I.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_gather_element_trace(hdgb_disc* d, const double* face_values, double* out) {
    hdgb_ctx* c = d->ctx;
    return guarded(c, [&] {
        const DiscView& v = d->view;
        InArg X(c, face_values, static_cast<size_t>(v.mpf) * v.nf);
        OutArg Y(c, out, static_cast<size_t>(v.nfl) * v.ne);
        launch_gather_element_trace(c, X.dev, v.elem_faces, v.ne, v.n_lfe, v.mpf, Y.dev);
        Y.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

hdgb_status hdgb_recover_local(hdgb_disc* d, const hdgb_ops* o, const double* duhat, double* du) {
    hdgb_ctx* c = d->ctx;
    return guarded(c, [&] {
        const DiscView& v = d->view;
        InArg X(c, duhat, static_cast<size_t>(v.mpf) * v.nf);
        OutArg Y(c, du, static_cast<size_t>(v.npe) * v.ne);
        DevBuf<double> tmp(static_cast<size_t>(v.npe) * v.ne);
        recover_local_device(d, o, X.dev, Y.dev, tmp.p);
        Y.commit();
        HDGB_CUDA(cudaStreamSynchronize(c->stream));
    });
}

}  // extern "C"
