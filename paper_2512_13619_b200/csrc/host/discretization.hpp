// Host-side setup layer ("mesh/master-element setup" of the reference API): quadrature rules,
// nodal bases tabulated at quadrature points, mesh connectivity with face orientations, and the
// geometric factors.  Setup-time, serial, host code -- the tables are uploaded once and consumed
// by the device kernels.  For 2D quadrilaterals the tables reproduce the reference's
// (basis.cpp, mesh.cpp) numbering and arithmetic, which tests check bit for bit against oracle/_ref.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "../../../include/hdgb200.h"

namespace hdgb {

struct Rule1D {
    std::vector<double> pts, wts;
    int size() const { return static_cast<int>(pts.size()); }
};

// Gauss-Legendre on [0,1], q points (basis.cpp:33-62 semantics: Newton on Legendre, symmetric).
Rule1D gauss_rule(int q);
// Gauss-Lobatto nodes on [0,1] (basis.cpp:79-104).
std::vector<double> lobatto_nodes(int n);
void lagrange_values(const std::vector<double>& nodes, double x, double* out);
void lagrange_derivs(const std::vector<double>& nodes, double x, double* out);

// Shape constants.
struct ShapeInfo {
    int dim;
    int n_lfe;     // local faces
    int vpe;       // vertices per element
    int vpf;       // vertices per face
    int n_orient;  // relative orientations of a face side
    // local face -> element-local vertex ids, listed in the face's local parameter corner order
    int face_verts[6][4];
    // +1 if (dX/ds x dX/dt) [3D] / tangent rotated by -90 degrees [2D] of the local face
    // parameterisation points outward, -1 otherwise
    int outward_sign[6];
};
const ShapeInfo& shape_info(int shape);

// The master element: everything tabulated on the reference element (generalised BasisTab,
// basis.hpp:44-67).
struct MasterElement {
    int shape = HDGB_QUAD, dim = 2, degree = 1;
    int pe = 0, pf = 0, qe = 0, qf = 0, n_lfe = 4, n_orient = 2;
    Rule1D rule1d;
    std::vector<double> nodes1d;
    std::vector<double> elem_pts;  // qe x dim reference points
    std::vector<double> elem_wts;  // qe
    std::vector<double> face_pts;  // qf x (dim-1) canonical face parameters
    std::vector<double> face_wts;  // qf
    std::vector<double> phi;       // pe x qe, [i + pe*g]
    std::array<std::vector<double>, 3> dphi;  // d/dxi_r, pe x qe each
    std::vector<double> psi;       // pf x qf, [l + pf*g]
    // element basis on local face lf seen with relative orientation o, at the CANONICAL face
    // quadrature point gc: tphi[((lf*n_orient + o)*qf + gc)*pe + i]
    std::vector<double> tphi;
    // un-oriented tables in the element-local face parameterisation (== reference trace_phi[lf])
    std::vector<double> tphi_local;  // [(lf*qf + g)*pe + i]
    // canonical -> side-local face quadrature index for each orientation: qperm[o*qf + gc]
    // (tensor shapes only: their symmetric rules map onto themselves; simplex tables are evaluated
    // directly at the mapped points)
    std::vector<int> qperm;
    std::vector<double> elem_nodes;  // pe x dim      reference coordinates of the nodal basis points
    std::vector<double> face_nodes;  // pf x (dim-1)  canonical face parameters of the trace nodes
};
MasterElement make_master_element(int shape, int degree, int quad_points);

// Mesh connectivity (generalised Mesh2D, mesh.hpp:24-39).
struct HostMesh {
    int shape = HDGB_QUAD, dim = 2;
    int ne = 0, nf = 0, nv = 0, n_lfe = 4, vpe = 4, vpf = 2;
    std::vector<int> elem_verts;   // ne x vpe
    std::vector<int> elem_faces;   // ne x n_lfe   (element_to_face)
    std::vector<int> face_elems;   // nf x 2       (face_to_elements, -1 on the boundary)
    std::vector<int> face_lidx;    // nf x 2       (face_local_index)
    std::vector<int> face_orient;  // nf x 2       (0 = canonical; 2D: 1 = reversed)
    std::vector<int> face_verts;   // nf x vpf     canonical corner order
    std::vector<int> bnd_tag;      // nf           0 interior
    std::vector<double> coords;    // nv x dim
    std::vector<int> elem_side;    // ne x n_lfe   which side of its face the element is (derived)
};
// Structured n^D mesh of the box; quads reproduce mesh.cpp:18-107 exactly.  TRI / TET split each
// cell (2 triangles / 6 Kuhn tetrahedra).  jitter displaces interior vertices.
HostMesh build_structured_mesh(int shape, int n, const double* lo, const double* hi, double jitter,
                               uint64_t seed);
// Generic conforming mesh from element vertex lists.
HostMesh build_mesh_from_elements(int shape, int ne, int nv, const int32_t* elem_verts,
                                  const double* coords);

// Mesh whose connectivity is given explicitly (sub-domain meshes cut out of a global mesh keep the
// global face orientations / side assignment).  face_elems entries < 0 mean "no local element on
// that side" (-1: domain boundary, -2: element lives on another rank).
HostMesh mesh_from_tables(int shape, int ne, int nf, int nv, const int32_t* elem_verts, const double* coords,
                          const int32_t* elem_faces, const int32_t* face_elems, const int32_t* face_lidx,
                          const int32_t* face_orient, const int32_t* face_verts, const int32_t* bnd_tag);

// Geometric factors at quadrature points (generalised GeomFactors, mesh.hpp:47-60).
struct HostGeom {
    std::vector<double> elem_detjac;  // [e*qe + g]
    std::vector<double> elem_invjac;  // [(e*qe + g)*D*D + r*D + c] = d xi_r / d x_c
    std::vector<double> elem_coords;  // [(e*qe + g)*D + c]
    std::vector<double> face_detjac;  // [f*qf + g]
    std::vector<double> face_coords;  // [(f*qf + g)*D + c]
    std::vector<double> face_normal;  // [((f*2 + side)*qf + g)*D + c], outward of that side
};
HostGeom compute_geometry(const HostMesh& mesh, const MasterElement& me);

}  // namespace hdgb
