// Element-local kernels: quadrature assembly of the weak residual and of the
// Jacobian blocks D_d, E, F, G_d, H, J (local_ops.cpp:33-228) and the state-independent factors
// M, B_d, C_d (local_ops.cpp:252-337).
//
// local_assemble: one CTA per element, two phases.
//   (1) point evaluation: threads sweep the qe volume and n_lfe*qf face quadrature points,
//       interpolate (u, q, uhat), evaluate the model functor and leave one coefficient record per
//       point in shared memory (the reference calls 8 std::function objects per point instead);
//   (2) contraction: threads own output entries and accumulate them over the points in the
//       reference's order (volume points ascending, then faces lf ascending, gc ascending), so
//       every entry sees the same sequence of terms as the reference (differences: FMA only).
// Roofline: FP64 pipe; per-element traffic is one write of the raw blocks.
#include "kernels_local.cuh"
#include "models.cuh"
#include "tma.cuh"

namespace hdgb {

namespace {

// ---- setup kernels ---------------------------------------------------------------------------------
// mass(i,j) = sum_g (phi_i phi_j)(g) * (w_g detJ_g)        (local_ops.cpp:266-281)
// bmat_d(i,j) = sum_g (w detJ phi_j)(g) * grad_d phi_i(g)   (local_ops.cpp:288-307)
// One CTA per element; the per-point weights and inverse Jacobians are staged once in shared memory and a
// thread owns a 2 x 4 tile of (i, j) pairs, so every table value loaded serves 4 (resp. 2) entries.  The terms of
// an entry are formed and summed exactly as in the scalar version (points ascending).
[[maybe_unused]] constexpr int kMbTi = 2, kMbTj = 4;
template <int D>
__global__ void __launch_bounds__(256) mass_bmat_kernel(DiscView dv, double* __restrict__ mass, double* __restrict__ b0,
                                                        double* __restrict__ b1, double* __restrict__ b2) {
    extern __shared__ double sm_setup[];
    const int e = blockIdx.x;
    const int pe = dv.pe, qe = dv.qe;
    double* sw = sm_setup;       // qe
    double* sj = sw + qe;        // qe * D * D
    for (int g = threadIdx.x; g < qe; g += blockDim.x) sw[g] = dv.wq[g] * dv.elem_detjac[static_cast<size_t>(e) * qe + g];
    for (int t = threadIdx.x; t < qe * D * D; t += blockDim.x) sj[t] = dv.elem_invjac[static_cast<size_t>(e) * qe * D * D + t];
    __syncthreads();
    const int nti = (pe + kMbTi - 1) / kMbTi, ntj = (pe + kMbTj - 1) / kMbTj;
    for (int t = threadIdx.x; t < nti * ntj; t += blockDim.x) {
        const int tj = t / nti, ti = t - tj * nti;
        int ii[kMbTi], jj[kMbTj];
#pragma unroll
        for (int a = 0; a < kMbTi; ++a) ii[a] = min(ti * kMbTi + a, pe - 1);
#pragma unroll
        for (int c = 0; c < kMbTj; ++c) jj[c] = min(tj * kMbTj + c, pe - 1);
        double am[kMbTi][kMbTj], ab[kMbTi][kMbTj][D];
#pragma unroll
        for (int a = 0; a < kMbTi; ++a)
#pragma unroll
            for (int c = 0; c < kMbTj; ++c) {
                am[a][c] = 0.0;
#pragma unroll
                for (int d = 0; d < D; ++d) ab[a][c][d] = 0.0;
            }
        for (int g = 0; g < qe; ++g) {
            const double w = sw[g];
            const double* ij = sj + g * D * D;
            double pi[kMbTi], gd[kMbTi][D], pj[kMbTj];
#pragma unroll
            for (int a = 0; a < kMbTi; ++a) {
                pi[a] = __ldg(dv.phi + ii[a] + pe * g);
                double dp[D];
#pragma unroll
                for (int r = 0; r < D; ++r) dp[r] = __ldg(dv.dphi[r] + ii[a] + pe * g);
#pragma unroll
                for (int d = 0; d < D; ++d) {
                    double s = 0.0;
#pragma unroll
                    for (int r = 0; r < D; ++r) s += dp[r] * ij[r * D + d];
                    gd[a][d] = s;
                }
            }
#pragma unroll
            for (int c = 0; c < kMbTj; ++c) pj[c] = __ldg(dv.phi + jj[c] + pe * g);
#pragma unroll
            for (int a = 0; a < kMbTi; ++a)
#pragma unroll
                for (int c = 0; c < kMbTj; ++c) {
                    am[a][c] += (pi[a] * pj[c]) * w;
                    const double wpj = w * pj[c];
#pragma unroll
                    for (int d = 0; d < D; ++d) ab[a][c][d] += wpj * gd[a][d];
                }
        }
#pragma unroll
        for (int a = 0; a < kMbTi; ++a)
#pragma unroll
            for (int c = 0; c < kMbTj; ++c) {
                const int i = ti * kMbTi + a, j = tj * kMbTj + c;
                if (i >= pe || j >= pe) continue;
                const size_t o = static_cast<size_t>(e) * pe * pe + static_cast<size_t>(j) * pe + i;
                mass[o] = am[a][c];
                b0[o] = ab[a][c][0];
                b1[o] = ab[a][c][1];
                if (D == 3) b2[o] = ab[a][c][D - 1];
            }
    }
}

// cmat_d(i, (lf,b)) = - sum_gc (w psi_b)(gc) * phis_i(gc) * n_d   (local_ops.cpp:310-336)
// Same scheme: per-face weights and normals staged in shared memory, a thread owns 2 (i) x 4 (b) entries of one
// local face.
template <int D>
__global__ void __launch_bounds__(256) cmat_kernel(DiscView dv, double* __restrict__ c0, double* __restrict__ c1, double* __restrict__ c2) {
    extern __shared__ double sm_setup[];
    const int e = blockIdx.x;
    const int pe = dv.pe, pf = dv.pf, qf = dv.qf, nfs = dv.nfs, n_lfe = dv.n_lfe;
    double* sw = sm_setup;              // n_lfe * qf
    double* sn = sw + n_lfe * qf;       // n_lfe * qf * D
    __shared__ int s_orient[8];
    if (threadIdx.x < n_lfe) {
        const int f = dv.elem_faces[e * n_lfe + threadIdx.x];
        s_orient[threadIdx.x] = dv.face_orient[2 * f + dv.elem_side[e * n_lfe + threadIdx.x]];
    }
    for (int t = threadIdx.x; t < n_lfe * qf; t += blockDim.x) {
        const int lf = t / qf, gc = t - lf * qf;
        const int f = dv.elem_faces[e * n_lfe + lf], side = dv.elem_side[e * n_lfe + lf];
        sw[t] = dv.wf[gc] * dv.face_detjac[static_cast<size_t>(f) * qf + gc];
        const double* n = dv.face_normal + ((static_cast<size_t>(f) * 2 + side) * qf + gc) * D;
#pragma unroll
        for (int d = 0; d < D; ++d) sn[t * D + d] = n[d];
    }
    __syncthreads();
    const int nti = (pe + kMbTi - 1) / kMbTi, ntb = (pf + kMbTj - 1) / kMbTj;
    for (int t = threadIdx.x; t < n_lfe * ntb * nti; t += blockDim.x) {
        const int lf = t / (ntb * nti), r2 = t - lf * (ntb * nti);
        const int tb = r2 / nti, ti = r2 - tb * nti;
        int ii[kMbTi], bb[kMbTj];
#pragma unroll
        for (int a = 0; a < kMbTi; ++a) ii[a] = min(ti * kMbTi + a, pe - 1);
#pragma unroll
        for (int c = 0; c < kMbTj; ++c) bb[c] = min(tb * kMbTj + c, pf - 1);
        const double* tp = dv.tphi + (static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf * pe;
        double acc[kMbTi][kMbTj][D];
#pragma unroll
        for (int a = 0; a < kMbTi; ++a)
#pragma unroll
            for (int c = 0; c < kMbTj; ++c)
#pragma unroll
                for (int d = 0; d < D; ++d) acc[a][c][d] = 0.0;
        for (int gc = 0; gc < qf; ++gc) {
            const double w = sw[lf * qf + gc];
            const double* n = sn + (lf * qf + gc) * D;
            double ph[kMbTi], pb[kMbTj];
#pragma unroll
            for (int a = 0; a < kMbTi; ++a) ph[a] = __ldg(tp + static_cast<size_t>(gc) * pe + ii[a]);
#pragma unroll
            for (int c = 0; c < kMbTj; ++c) pb[c] = w * __ldg(dv.psi + bb[c] + pf * gc);
#pragma unroll
            for (int a = 0; a < kMbTi; ++a)
#pragma unroll
                for (int c = 0; c < kMbTj; ++c)
#pragma unroll
                    for (int d = 0; d < D; ++d) acc[a][c][d] -= pb[c] * ph[a] * n[d];
        }
#pragma unroll
        for (int a = 0; a < kMbTi; ++a)
#pragma unroll
            for (int c = 0; c < kMbTj; ++c) {
                const int i = ti * kMbTi + a, b = tb * kMbTj + c;
                if (i >= pe || b >= pf) continue;
                const size_t off = static_cast<size_t>(e) * pe * nfs + static_cast<size_t>(lf * pf + b) * pe + i;
                c0[off] = acc[a][c][0];
                c1[off] = acc[a][c][1];
                if (D == 3) c2[off] = acc[a][c][D - 1];
            }
    }
}

// ---- the assembly kernel -------------------------------------------------------------------------------
// Point records keep the model coefficients already contracted with the inverse Jacobian
// (index r = reference direction), so that the basis contraction needs d(phi_i)/d(xi_r) only:
//   sum_d C_d * grad_d(phi_i) = sum_r dphi_r,i * (sum_d invj[r][d] * C_d).
template <int M, int D>
struct VolRec {
    double w;
    double Fr[M * D];          // [m*D + r]
    double S[M];
    double tm[M];              // dt_inv * (u - u_prev)
    double cE[M * M * D];      // [(m*M + mp)*D + r]          from dF/du
    double dSu[M * M];
    double cD[D * M * M * D];  // [((dp*M + m)*M + mp)*D + r] from dF/dq_dp
    double dSq[M * M * D];
};

template <int M, int D>
struct FaceRec {
    double w;
    double fhat[M];
    double val[M];
    double tau;
    double dfh_q[M * M * D];
    double dfh_uh[M * M];
    double dv_u[M * M];
    double dv_q[M * M * D];
    double dv_uh[M * M];
};

// ---- E and D_d on the FP64 tensor-core path -----------------------------------------------------------
// For one component pair (m, mp) the 1 + D blocks E[(m,.),(mp,.)], D_dp[(m,.),(mp,.)] are
//     X_w[i, j] = sum_pts V_w[i, pt] * (w_pt phi_j(pt)),   w = 0 (E), 1 + dp (D_dp),
// with the volume points followed by the face points as the contraction index: a batch of
// (pe x npts) x (npts x pe) products sharing their right operand.  The points are swept in chunks of
// 16; per chunk the CTA builds V_w (point coefficients x basis tables, a few FMAs per entry) and the
// weighted basis in shared memory and every warp multiplies its 16 x 32 output tiles with DMMA
// m8n8k4.  Several component pairs are processed per pass when pe is small.  Summation order: points
// in groups of 4 inside the tensor core (reference: strictly ascending), equal to rounding.
__device__ __forceinline__ void dmma_8x8x4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

constexpr int kResParts = 8;   // thread groups sharing one basis function's point sweep in the residual phase
constexpr int kEdKc = 16;      // points per chunk
constexpr int kEdSlotsMax = 4;  // 16 x 32 output tiles per warp: 2 for scalar systems (two CTAs per SM), 4 for wide ones (fewer passes)
__host__ __device__ constexpr int ed_slots(int M) { return M == 1 ? 2 : kEdSlotsMax; }

// Operand chunks are stored POINT-major ([point in chunk][basis function], leading dimensions = 4 mod 16): the
// builder's half-warps write 16 consecutive basis functions of one point (conflict-free stores) and both DMMA
// fragment loads -- A: (row grp, k tig) -> [k][row], B: (k tig, column grp) -> [k][column] -- hit 16 distinct
// 8-byte banks per half-warp.
struct EdPlan {
    int rg, cg;   // 16-row / 32-column tile groups covering pe
    int pp;       // component pairs per pass
    int lda;      // leading dimension of a V_w chunk (= 4 mod 16)
    int ldb;      // leading dimension of the weighted-basis chunk (= 4 mod 16)
    int wsub;     // V_w matrices resident per sub-pass (the warps' accumulator slots cover that many at a time)
    __host__ __device__ size_t doubles(int D) const {
        return static_cast<size_t>(wsub) * kEdKc * lda + static_cast<size_t>(kEdKc) * ldb;
    }
};
inline __host__ __device__ EdPlan ed_plan(int pe, int M, int D, int nwarps) {
    const int kEdSlots = ed_slots(M);
    EdPlan p;
    p.rg = (pe + 15) / 16;
    p.cg = (pe + 31) / 32;
    p.lda = p.rg * 16 + 4;
    p.ldb = p.cg * 32 + 4;
    const int per_pair = (1 + D) * p.rg * p.cg;
    const int gs = nwarps * kEdSlots, rc = p.rg * p.cg;  // gs: 16 x 32 tiles the CTA's accumulator slots hold at a time
    int pp = gs / per_pair;                               // component pairs sharing one sweep (and one weighted basis)
    if (pp < 1) pp = 1;
    if (pp > M * M) pp = M * M;
    p.pp = pp;
    const int qp = pp * (1 + D);
    int wsub = (gs + rc - 1) / rc + ((gs % rc) ? 1 : 0);
    if (wsub > qp) wsub = qp;
    p.wsub = wsub;
    return p;
}
// usable when one pass's tiles fit the warps' accumulator slots
inline bool ed_dmma_ok(int pe, int M, int D) { return pe <= 64 && pe >= tuning().local_dmma_min_pe; }


// Point records in the global scratch (GREC) are read with ld.global.cg: an explicit global-space load that the
// compiler may hoist above the shared-memory stores of the operand builder (a generic load may not be), coherent
// at L2 with the records this CTA wrote earlier in the kernel.
template <bool GREC>
__device__ __forceinline__ double rec_ld(const double* p) {
    if constexpr (GREC) return __ldcg(p);
    else return *p;
}

template <int M, int D, bool GREC>
__device__ void ed_dmma(const DiscView& dv, const LocalIn& in, const LocalOut& out, int e, const VolRec<M, D>* vrec,
                        const FaceRec<M, D>* frec, const int* s_orient, double* opbuf, int gv0, int gv1, int fp0, int fp1,
                        int first) {
    // vrec / frec hold the records of volume points [gv0, gv1) and face points [fp0, fp1) (one chunk of a
    // point-chunked sweep, or all points); later chunks accumulate into the blocks (first == 0)
    constexpr int kEdSlots = ed_slots(M);
    constexpr int kEdRes = (M == 1) ? 2 : 4;  // resident matrices whose coefficient rows the cached builder keeps in registers
    constexpr int kEdIt = 4;                  // strips of 16 basis functions covering the padded columns (pe <= 64)
    // Table loads of the next chunk issued before the current chunk's products, operands finished after them: pays
    // where the registers are there (one CTA per SM, 255 registers: config 5 local kernel 37.0 -> 35.5 ms at hex 12^3);
    // at two CTAs per SM (128 registers) the 16 prefetched values spill and the kernel loses (17.2 -> 19.0 ms at config 2).
    constexpr bool kSplitBuild = GREC;
    const int pe = dv.pe, qf = dv.qf, npe = M * pe;
    const int qe = gv1 - gv0, nfp = fp1 - fp0;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const EdPlan pl = ed_plan(pe, M, D, nwarps);
    const int lda = pl.lda;
    const int bufd = static_cast<int>(pl.doubles(D));  // one operand buffer: [wsub][kc][lda] then [kc][ldb]; two of them
    const int boff0 = pl.wsub * kEdKc * lda;
    const int rc = pl.rg * pl.cg;
    const bool transient = in.dt_inv > 0.0;
    const int gpp = (1 + D) * pl.rg * pl.cg;  // tile groups per component pair
    const int nchunk_v = (qe + kEdKc - 1) / kEdKc, nchunk_f = (nfp + kEdKc - 1) / kEdKc;
    const int nchunk = nchunk_v + nchunk_f;

    // Builder mapping (blockDim.x == 256 = 16 half-warps): half-warp <-> point of the chunk, lanes <-> basis functions
    // i0, i0 + 16, ...  A thread reads its point's coefficients once per chunk and the basis tables with 128-byte
    // half-warp loads; every operand entry the products read (incl. the zero padding) is written by exactly one thread.
    // With 512 threads two half-warps share a point: each builds every second resident matrix (cached builder only).
    const int bkk = (tid >> 4) & 15, bi0 = tid & 15, bsub = tid >> 8, nsub = nt >> 8;
    const int irows = pl.rg * 16, icols = pl.cg * 32, ldb = pl.ldb;
    for (int pair0 = 0; pair0 < M * M; pair0 += pl.pp) {
        const int npair = min(pl.pp, M * M - pair0);
        const int ngroups = npair * gpp;
        int wlo = 0, whi = npair * (1 + D);  // V_w matrices of the current sub-pass
        // chunk builder: V_w and the weighted basis of points [p0, p0 + 16) into operand buffer `buf`
        auto build = [&](int ch, int buf) {
            double* Ab = opbuf + buf * bufd;
            double* Bb = Ab + boff0;
            const bool vol = ch < nchunk_v;
            const int p0 = vol ? ch * kEdKc : (ch - nchunk_v) * kEdKc;
            const int np = min(kEdKc, (vol ? qe : nfp) - p0);
            const bool live = bkk < np;
            const int pt = live ? p0 + bkk : 0;
            if (vol) {
                const int g = gv0 + pt;
                const VolRec<M, D>& r = vrec[pt];
                const double wq = live ? rec_ld<GREC>(&r.w) : 0.0;
                const double* php = dv.phi + static_cast<size_t>(pe) * g;
                const double* dpp[D];
#pragma unroll
                for (int k = 0; k < D; ++k) dpp[k] = dv.dphi[k] + static_cast<size_t>(pe) * g;
                for (int pi = 0; pi < npair; ++pi) {
                    const int pr = pair0 + pi, mp = pr / M, m = pr - mp * M, mm = m * M + mp;
                    const int w0 = pi * (1 + D);
                    // coefficient rows of this pair's matrices that are resident in the sub-pass
                    bool on[1 + D];
                    double cph[1 + D], cdp[1 + D][D];
#pragma unroll
                    for (int w = 0; w <= D; ++w) {
                        on[w] = w0 + w >= wlo && w0 + w < whi;
                        cph[w] = 0.0;
#pragma unroll
                        for (int k = 0; k < D; ++k) cdp[w][k] = 0.0;
                    }
                    if (on[0]) {
                        cph[0] = rec_ld<GREC>(&r.dSu[mm]);
#pragma unroll
                        for (int k = 0; k < D; ++k) cdp[0][k] = rec_ld<GREC>(&r.cE[mm * D + k]);
                    }
#pragma unroll
                    for (int dq = 0; dq < D; ++dq)
                        if (on[1 + dq]) {
                            cph[1 + dq] = rec_ld<GREC>(&r.dSq[mm * D + dq]);
#pragma unroll
                            for (int k = 0; k < D; ++k) cdp[1 + dq][k] = rec_ld<GREC>(&r.cD[(dq * M * M + mm) * D + k]);
                        }
                    const bool tdiag = transient && m == mp;
                    for (int i = bi0; i < icols; i += 16) {
                        const bool inb = live && i < pe;  // outside: exact zero padding
                        const double ph = inb ? __ldg(php + i) : 0.0;
                        double dp_[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) dp_[k] = inb ? __ldg(dpp[k] + i) : 0.0;
                        if (i < irows) {
#pragma unroll
                            for (int w = 0; w <= D; ++w) {
                                if (!on[w]) continue;
                                double fs = 0.0;
#pragma unroll
                                for (int k = 0; k < D; ++k) fs += cdp[w][k] * dp_[k];
                                double v = -fs - cph[w] * ph;
                                if (w == 0 && tdiag) v += in.dt_inv * ph;
                                Ab[((w0 + w - wlo) * kEdKc + bkk) * lda + i] = inb ? v : 0.0;
                            }
                        }
                        if (pi == 0) Bb[bkk * ldb + i] = wq * ph;
                    }
                }
            } else {
                const int p = fp0 + pt;
                const int lf = p / qf, gc = p - lf * qf;
                const FaceRec<M, D>& r = frec[pt];
                const double wq = live ? rec_ld<GREC>(&r.w) : 0.0;
                const double* php = dv.tphi + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe;
                for (int pi = 0; pi < npair; ++pi) {
                    const int pr = pair0 + pi, mp = pr / M, m = pr - mp * M, mm = m * M + mp;
                    const int w0 = pi * (1 + D);
                    bool on[1 + D];
                    double cf[1 + D];
#pragma unroll
                    for (int w = 0; w <= D; ++w) {
                        on[w] = w0 + w >= wlo && w0 + w < whi;
                        cf[w] = 0.0;
                    }
                    if (on[0] && m == mp) cf[0] = rec_ld<GREC>(&r.tau);
#pragma unroll
                    for (int dq = 0; dq < D; ++dq)
                        if (on[1 + dq]) cf[1 + dq] = rec_ld<GREC>(&r.dfh_q[mm * D + dq]);
                    for (int i = bi0; i < icols; i += 16) {
                        const bool inb = live && i < pe;
                        const double ph = inb ? __ldg(php + i) : 0.0;
                        if (i < irows) {
#pragma unroll
                            for (int w = 0; w <= D; ++w)
                                if (on[w]) Ab[((w0 + w - wlo) * kEdKc + bkk) * lda + i] = inb ? cf[w] * ph : 0.0;
                        }
                        if (pi == 0) Bb[bkk * ldb + i] = wq * ph;
                    }
                }
            }
        };
        // The same builder with everything hoisted for the common shapes (the resident matrices of a sub-pass fit
        // kEdRes coefficient rows in registers: scalar systems with pe in 49..64, wide systems one pair per pass):
        // coefficient rows read once per chunk, the basis-function strips unrolled with constant offsets.
        // Stage 1 of the cached builder: only the table loads of chunk ch (this thread's point, its strips of 16 basis
        // functions) -- issued BEFORE the products of the current chunk so that their L2 latency is covered by the
        // warp's own DMMA chain; stage 2 (coefficient rows from the records, FMAs, shared-memory stores) runs after it.
        auto load_tables = [&](int ch, double (&tb)[kEdIt][1 + D]) {
            const bool vol = ch < nchunk_v;
            const int p0 = vol ? ch * kEdKc : (ch - nchunk_v) * kEdKc;
            const int np = min(kEdKc, (vol ? qe : nfp) - p0);
            const bool live = bkk < np;
            const int pt = live ? p0 + bkk : 0;
            if (vol) {
                const int g = gv0 + pt;
                const double* php = dv.phi + static_cast<size_t>(pe) * g + bi0;
                const double* dpp[D];
#pragma unroll
                for (int k = 0; k < D; ++k) dpp[k] = dv.dphi[k] + static_cast<size_t>(pe) * g + bi0;
#pragma unroll
                for (int it = 0; it < kEdIt; ++it) {
                    const bool inb = live && 16 * it < icols && bi0 + 16 * it < pe;  // outside: exact zero padding
                    tb[it][0] = inb ? __ldg(php + 16 * it) : 0.0;
#pragma unroll
                    for (int k = 0; k < D; ++k) tb[it][1 + k] = inb ? __ldg(dpp[k] + 16 * it) : 0.0;
                }
            } else {
                const int p = fp0 + pt;
                const int lf = p / qf, gc = p - lf * qf;
                const double* php = dv.tphi + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe + bi0;
#pragma unroll
                for (int it = 0; it < kEdIt; ++it) {
                    const bool inb = live && 16 * it < icols && bi0 + 16 * it < pe;
                    tb[it][0] = inb ? __ldg(php + 16 * it) : 0.0;
                }
            }
        };
        auto build_cached = [&](int ch, int buf, const double (&tb)[kEdIt][1 + D]) {
            double* Ab = opbuf + buf * bufd + bkk * lda + bi0;       // this thread's entry of resident matrix 0, strip 0
            double* Bb = opbuf + buf * bufd + boff0 + bkk * ldb + bi0;
            const bool vol = ch < nchunk_v;
            const int p0 = vol ? ch * kEdKc : (ch - nchunk_v) * kEdKc;
            const int np = min(kEdKc, (vol ? qe : nfp) - p0);
            const bool live = bkk < np;
            const int pt = live ? p0 + bkk : 0;
            const int nres = whi - wlo;
            const int qstride = kEdKc * lda;
            // this thread's resident matrices: q = bsub, bsub + nsub, ... (kEdRes of them at most)
            if (vol) {
                const VolRec<M, D>& r = vrec[pt];
                const double wq = rec_ld<GREC>(&r.w);
                double c0[kEdRes], ck[kEdRes][D];
                bool td[kEdRes];
#pragma unroll
                for (int qi = 0; qi < kEdRes; ++qi) {
                    const int q = bsub + nsub * qi;
                    c0[qi] = 0.0;
                    td[qi] = false;
#pragma unroll
                    for (int k = 0; k < D; ++k) ck[qi][k] = 0.0;
                    if (q < nres) {
                        const int wg = wlo + q, pi = wg / (1 + D), w = wg - pi * (1 + D);
                        const int pr = pair0 + pi, mp = pr / M, m = pr - mp * M, mm = m * M + mp;
                        if (w == 0) {
                            c0[qi] = rec_ld<GREC>(&r.dSu[mm]);
#pragma unroll
                            for (int k = 0; k < D; ++k) ck[qi][k] = rec_ld<GREC>(&r.cE[mm * D + k]);
                            td[qi] = transient && m == mp;
                        } else {
                            c0[qi] = rec_ld<GREC>(&r.dSq[mm * D + w - 1]);
#pragma unroll
                            for (int k = 0; k < D; ++k) ck[qi][k] = rec_ld<GREC>(&r.cD[((w - 1) * M * M + mm) * D + k]);
                        }
                    }
                }
                const double* php = dv.phi + static_cast<size_t>(pe) * (gv0 + pt) + bi0;
                const double* dpp[D];
#pragma unroll
                for (int k = 0; k < D; ++k) dpp[k] = dv.dphi[k] + static_cast<size_t>(pe) * (gv0 + pt) + bi0;
#pragma unroll
                for (int it = 0; it < kEdIt; ++it) {
                    if (16 * it >= icols) break;
                    const bool inb = live && bi0 + 16 * it < pe;
                    // prefetched by load_tables (split build) or loaded here, strip by strip
                    const double ph = kSplitBuild ? tb[it][0] : (inb ? __ldg(php + 16 * it) : 0.0);
                    double dp_[D];
#pragma unroll
                    for (int k = 0; k < D; ++k) dp_[k] = kSplitBuild ? tb[it][1 + k] : (inb ? __ldg(dpp[k] + 16 * it) : 0.0);
                    if (16 * it < irows) {
#pragma unroll
                        for (int qi = 0; qi < kEdRes; ++qi) {
                            const int q = bsub + nsub * qi;
                            if (q >= nres) break;
                            double fs = 0.0;
#pragma unroll
                            for (int k = 0; k < D; ++k) fs += ck[qi][k] * dp_[k];
                            double v = -fs - c0[qi] * ph;
                            if (td[qi]) v += in.dt_inv * ph;
                            Ab[q * qstride + 16 * it] = inb ? v : 0.0;
                        }
                    }
                    if (bsub == 0) Bb[16 * it] = inb ? wq * ph : 0.0;
                }
            } else {
                const FaceRec<M, D>& r = frec[pt];
                const double wq = rec_ld<GREC>(&r.w);
                double cf[kEdRes];
#pragma unroll
                for (int qi = 0; qi < kEdRes; ++qi) {
                    const int q = bsub + nsub * qi;
                    cf[qi] = 0.0;
                    if (q < nres) {
                        const int wg = wlo + q, pi = wg / (1 + D), w = wg - pi * (1 + D);
                        const int pr = pair0 + pi, mp = pr / M, m = pr - mp * M, mm = m * M + mp;
                        if (w == 0) cf[qi] = (m == mp) ? rec_ld<GREC>(&r.tau) : 0.0;
                        else cf[qi] = rec_ld<GREC>(&r.dfh_q[mm * D + w - 1]);
                    }
                }
                const int pf_ = fp0 + pt;
                const int lf = pf_ / qf, gc = pf_ - lf * qf;
                const double* php = dv.tphi + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe + bi0;
#pragma unroll
                for (int it = 0; it < kEdIt; ++it) {
                    if (16 * it >= icols) break;
                    const bool inb = live && bi0 + 16 * it < pe;
                    const double ph = kSplitBuild ? tb[it][0] : (inb ? __ldg(php + 16 * it) : 0.0);
                    if (16 * it < irows) {
#pragma unroll
                        for (int qi = 0; qi < kEdRes; ++qi) {
                            const int q = bsub + nsub * qi;
                            if (q >= nres) break;
                            Ab[q * qstride + 16 * it] = inb ? cf[qi] * ph : 0.0;
                        }
                    }
                    if (bsub == 0) Bb[16 * it] = inb ? wq * ph : 0.0;
                }
            }
        };
        for (int g0 = 0; g0 < ngroups; g0 += nwarps * kEdSlots) {  // sub-passes when the CTA has fewer warps than tiles
            wlo = g0 / rc;
            whi = (min(g0 + nwarps * kEdSlots, ngroups) - 1) / rc + 1;
            double acc[kEdSlots][2][4][2];
#pragma unroll
            for (int s = 0; s < kEdSlots; ++s)
#pragma unroll
                for (int a = 0; a < 2; ++a)
#pragma unroll
                    for (int b = 0; b < 4; ++b) acc[s][a][b][0] = acc[s][a][b][1] = 0.0;
            // tile coordinates of this warp's accumulator slots (fixed over the point sweep)
            int aoff[kEdSlots], boff[kEdSlots];
#pragma unroll
            for (int s = 0; s < kEdSlots; ++s) {
                const int gid = g0 + warp + nwarps * s;
                const int w = gid / (pl.rg * pl.cg), rem = gid - w * (pl.rg * pl.cg);
                const int rgi = rem / pl.cg, cgi = rem - rgi * pl.cg;
                aoff[s] = gid < ngroups ? (w - wlo) * kEdKc * lda + rgi * 16 + grp + tig * lda : -1;
                boff[s] = boff0 + cgi * 32 + grp + tig * ldb;
            }
            const bool cached = whi - wlo <= kEdRes * nsub;  // (the launcher uses 512 threads only where this holds)
            double tb[kEdIt][1 + D];  // prefetched table values of the next chunk (cached builder)
            __syncthreads();
            if (cached) {
                if (kSplitBuild) load_tables(0, tb);
                build_cached(0, 0, tb);
            } else {
                build(0, 0);
            }
            __syncthreads();
            for (int ch = 0; ch < nchunk; ++ch) {
                const int buf = ch & 1;
                // the next chunk's operands are built in the same barrier interval as this chunk's products:
                // warps drift apart, so table loads and DMMA issue overlap across the CTA
                if (ch + 1 < nchunk) {
                    if (cached) {
                        if (kSplitBuild) load_tables(ch + 1, tb);
                        else build_cached(ch + 1, buf ^ 1, tb);
                    } else {
                        build(ch + 1, buf ^ 1);
                    }
                }
                const double* Ob = opbuf + buf * bufd;
#pragma unroll
                for (int s = 0; s < kEdSlots; ++s) {
                    if (aoff[s] >= 0) {
                        const double* as = Ob + aoff[s];
                        const double* bs = Ob + boff[s];
#pragma unroll
                        for (int kk = 0; kk < kEdKc; kk += 4) {
                            double af[2], bf[4];
#pragma unroll
                            for (int a = 0; a < 2; ++a) af[a] = as[kk * lda + a * 8];
#pragma unroll
                            for (int b = 0; b < 4; ++b) bf[b] = bs[kk * ldb + b * 8];
#pragma unroll
                            for (int a = 0; a < 2; ++a)
#pragma unroll
                                for (int b = 0; b < 4; ++b) dmma_8x8x4(acc[s][a][b][0], acc[s][a][b][1], af[a], bf[b]);
                        }
                    }
                }
                // stage 2 of the cached builder: the tables requested before the products have arrived by now
                if (kSplitBuild && cached && ch + 1 < nchunk) build_cached(ch + 1, buf ^ 1, tb);
                __syncthreads();
            }
            // ---- write this pass's blocks ----
#pragma unroll
            for (int s = 0; s < kEdSlots; ++s) {
                const int gid = g0 + warp + nwarps * s;
                if (gid >= ngroups) continue;
                const int w = gid / (pl.rg * pl.cg), rem = gid - w * (pl.rg * pl.cg);
                const int rgi = rem / pl.cg, cgi = rem - rgi * pl.cg;
                const int pi = w / (1 + D), which = w - pi * (1 + D);
                const int pr = pair0 + pi, mp = pr / M, m = pr - mp * M;
                double* dst = (which == 0 ? out.E : out.Dm[which - 1]) + static_cast<size_t>(e) * npe * npe;
#pragma unroll
                for (int b = 0; b < 4; ++b)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int j = cgi * 32 + b * 8 + 2 * tig + h;
                        if (j >= pe) continue;
#pragma unroll
                        for (int a = 0; a < 2; ++a) {
                            const int i = rgi * 16 + a * 8 + grp;
                            if (i < pe) {
                                double* o = dst + static_cast<size_t>(mp * pe + j) * npe + (m * pe + i);
                                *o = first ? acc[s][a][b][h] : *o + acc[s][a][b][h];
                            }
                        }
                    }
            }
        }
    }
}

// ---- E and D_d of scalar systems with pe = 64: table ring + fragment-built operands ---------------------------
// The chunked builder above spends its time in dependent latency: table loads from L2 -> FMAs -> shared-memory
// stores -> CTA barrier -> fragment loads, once per 16 points.  For the hot shape (hex p = 3, M = 1)
// the sweep is restructured so that no operand is ever built in shared memory and no CTA barrier is taken:
//   * the basis tables of 8 points (phi, dphi_r rows of pe = 64 doubles, contiguous in global memory) are streamed by
//     bulk-TMA row copies into a 3-stage shared-memory ring ([table][point][68]: k-major, leading dimension = 4 mod 16,
//     conflict-free for both fragment loads); warp 0's lanes issue one row copy each, full / empty mbarriers per stage;
//   * warp w owns the 8 rows i = 8 w .. 8 w + 7 of TWO of the 1 + D matrices over all 64 columns (16 accumulator
//     tiles = the 128-register budget of two CTAs per SM); two sub-passes over the point list cover E, D_0 | D_1, D_2;
//   * per k-step of 4 points a lane reads ITS (row, point) entry of the 1 + D tables, forms the left fragment
//     a_w = -w_pt (c0_w phi + sum_r ck_w[r] dphi_r) of both resident matrices in registers from its point's
//     record (4 distinct records per warp: broadcast loads) and multiplies with the raw phi rows as right operand.
// Dead points of a partial stage copy a valid row (finite values) and get weight zero.  Same contraction as ed_dmma
// with the quadrature weight on the left operand instead of the right one: equal to rounding.
constexpr int kEsPts = 8;      // points per ring stage (two k-steps)
constexpr int kEsStages = 3;
constexpr int kEsLd = 68;      // 64 rows + 4
constexpr int kEsPe = 64;
inline __host__ __device__ size_t ed_stream_doubles(int D) { return static_cast<size_t>(kEsStages) * (1 + D) * kEsPts * kEsLd; }
inline bool ed_stream_ok(const DiscView& dv, int M) { return M == 1 && dv.D == 3 && dv.pe == kEsPe && dv.es_vol && (tuning().local_ed_stream & 3); }

template <int D>
__device__ void ed_stream(const DiscView& dv, const LocalIn& in, const LocalOut& out, int e, const VolRec<1, D>* vrec,
                          const FaceRec<1, D>* frec, const int* s_orient, double* ring, uint64_t* bars, bool do_ed, bool do_hgf, bool split_copies) {
    constexpr int NQ = 2;                       // resident matrices per sub-pass
    constexpr int NSP = (1 + D + NQ - 1) / NQ;  // sub-passes
    constexpr int NCT = kEsPe / 8;              // column tiles
    constexpr int stage_d = (1 + D) * kEsPts * kEsLd;
        const int qe = dv.qe, qf = dv.qf, nfp = dv.n_lfe * qf;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const int nsv = (qe + kEsPts - 1) / kEsPts, nsf = (nfp + kEsPts - 1) / kEsPts, nst = nsv + nsf;
    const int n_ed = do_ed ? NSP * nst : 0;            // E / D_d stages, then one stage per local face (H, G_d, F, J)
    const int hks = (qf + 3) / 4;                      // k-steps of a face stage
    const int total = n_ed + (do_hgf ? dv.n_lfe : 0);
    uint64_t* full = bars;
    uint64_t* empty = bars + kEsStages;
    const double dtv = in.dt_inv > 0.0 ? in.dt_inv : 0.0;

    // producer side (lane 0 of warp 0): stage s of a sub-pass into ring slot `slot`.  The padded stage images of the
    // volume tables (DiscView::es_vol, one contiguous block per stage) and the padded trace-table rows (es_face)
    // are prepared once per discretisation, so a stage is ONE bulk copy (volume) or one per local face it touches.
    auto issue = [&](int gi, int slot) {
        if (lane != 0) return;
        double* dst = ring + slot * stage_d;
        if (gi >= n_ed) {  // face stage: all points of local face gi - n_ed (rows past qf: the table's next rows, weight zero)
            const int lf = gi - n_ed;
            const uint32_t bytes = 4 * hks * kEsLd * sizeof(double);
            mbar_expect_tx(full + slot, bytes);
            const double* src = dv.es_face + (static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf * kEsLd;
            if (split_copies) {  // (measurement / sanitizer aid: copies of 4 rows)
                for (int r = 0; r < 4 * hks; r += 4) tma_bulk_g2s(dst + r * kEsLd, src + r * kEsLd, 4 * kEsLd * sizeof(double), full + slot);
            } else {
                tma_bulk_g2s(dst, src, bytes, full + slot);
            }
            return;
        }
        const int s = gi % nst;
        if (s < nsv) {
            mbar_expect_tx(full + slot, stage_d * sizeof(double));
            const double* src = dv.es_vol + static_cast<size_t>(s) * stage_d;
            if (split_copies) {
                for (int r = 0; r < (1 + D) * kEsPts; r += 4) tma_bulk_g2s(dst + r * kEsLd, src + r * kEsLd, 4 * kEsLd * sizeof(double), full + slot);
            } else {
                tma_bulk_g2s(dst, src, stage_d * sizeof(double), full + slot);
            }
        } else {
            constexpr uint32_t rb = kEsLd * sizeof(double);
            mbar_expect_tx(full + slot, kEsPts * rb);
            const int p0 = (s - nsv) * kEsPts;
            int p = p0;
            while (p < p0 + kEsPts) {
                const int pc = min(p, nfp - 1);  // dead points of the last stage: the last row again (finite values)
                const int lf = pc / qf, gc = pc - lf * qf;
                const int run = p < nfp ? min(min(p0 + kEsPts, nfp), (lf + 1) * qf) - p : 1;
                const double* src = dv.es_face + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * kEsLd;
                tma_bulk_g2s(dst + (p - p0) * kEsLd, src, run * rb, full + slot);
                p += run;
            }
        }
    };
    __syncthreads();  // earlier users of the ring's shared memory (generic proxy) are done
    if (warp == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int it = 0; it < kEsStages - 1 && it < total; ++it) issue(it, it);
    }

    double acc[NQ][NCT][2];
#pragma unroll
    for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int b = 0; b < NCT; ++b) acc[q][b][0] = acc[q][b][1] = 0.0;

    const int rowoff = 8 * warp + grp;  // this lane's row of the left fragments
    int slot = 0, par = 0;              // ring slot and parity of the stage being consumed
    int it = 0;
    // warp 0 keeps the ring kEsStages - 1 stages ahead of its own position
    auto produce = [&]() {
        if (warp != 0) return;
        const int nx = it + kEsStages - 1;
        if (nx < total) {
            int nslot = slot + kEsStages - 1;
            if (nslot >= kEsStages) nslot -= kEsStages;
            // the slot was last used by stage it - 1: wait until every warp released it
            if (it >= 1) mbar_wait(empty + nslot, ((it - 1) / kEsStages) & 1);
            issue(nx, nslot);
        }
    };
#pragma unroll
    for (int sp = 0; sp < (do_ed ? NSP : 0); ++sp) {
        const int w0 = sp * NQ;  // resident matrices w0, w0 + 1 (0 = E, 1 + d = D_d)
        for (int s = 0; s < nst; ++s, ++it) {
            produce();
            mbar_wait(full + slot, par);
            const double* St = ring + slot * stage_d;
            const bool vol = s < nsv;
            const int p0 = vol ? s * kEsPts : (s - nsv) * kEsPts;
            const int npts = vol ? qe : nfp;
#pragma unroll
            for (int ks = 0; ks < kEsPts / 4; ++ks) {
                const int p = 4 * ks + tig;
                const bool live = p0 + p < npts;
                const int pt = live ? p0 + p : npts - 1;
                double a[NQ];
                if (vol) {
                    const VolRec<1, D>& r = vrec[pt];
                    const double nw = live ? -r.w : 0.0;
                    const double t0 = St[p * kEsLd + rowoff];
                    double tk[D];
#pragma unroll
                    for (int k = 0; k < D; ++k) tk[k] = St[((1 + k) * kEsPts + p) * kEsLd + rowoff];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const int w = w0 + q;
                        if (w > D) { a[q] = 0.0; continue; }
                        double c0;
                        const double* ck;
                        if (w == 0) { c0 = r.dSu[0] - dtv; ck = r.cE; }
                        else { c0 = r.dSq[w - 1]; ck = r.cD + (w - 1) * D; }
                        double v = c0 * t0;
#pragma unroll
                        for (int k = 0; k < D; ++k) v = fma(ck[k], tk[k], v);
                        a[q] = nw * v;
                    }
                } else {
                    const FaceRec<1, D>& r = frec[pt];
                    const double wq = live ? r.w : 0.0;
                    const double t0 = wq * St[p * kEsLd + rowoff];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const int w = w0 + q;
                        a[q] = w > D ? 0.0 : (w == 0 ? r.tau : r.dfh_q[w - 1]) * t0;
                    }
                }
                const double* bs = St + p * kEsLd + grp;
#pragma unroll
                for (int b = 0; b < NCT; ++b) {
                    const double bf = bs[8 * b];
#pragma unroll
                    for (int q = 0; q < NQ; ++q)
                        if (w0 + q <= D) dmma_8x8x4(acc[q][b][0], acc[q][b][1], a[q], bf);
                }
            }
            ring_release_all(empty + slot);
            if (++slot == kEsStages) { slot = 0; par ^= 1; }
        }
        // ---- this sub-pass's blocks ----
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const int w = w0 + q;
            if (w > D) continue;
            double* dst = (w == 0 ? out.E : out.Dm[w - 1]) + static_cast<size_t>(e) * kEsPe * kEsPe + rowoff;
#pragma unroll
            for (int b = 0; b < NCT; ++b)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    dst[static_cast<size_t>(8 * b + 2 * tig + h) * kEsPe] = acc[q][b][h];
                    acc[q][b][h] = 0.0;
                }
        }
    }
    if (!do_hgf) return;
    // ---- H, G_d, F and J, one ring stage per local face (local_ops.cpp:186-219) ----
    //   [H | G_d](lf b, j) = sum_gc psi_b(gc) (cw(gc) phis_j(gc)),   F(i, lf bp) = sum_gc phis_i(gc) (cf(gc) psi_bp(gc)),
    //   J(lf b, lf bp)     = sum_gc psi_b(gc) (cj(gc) psi_bp(gc)).
    // psi (pf = 16 rows, the same for every face and element) lives in registers: lane (grp, tig) holds psi_{8 t + grp}(4 ks + tig),
    // which is both the left fragment of H / G_d / J and the right fragment of F / J.  The warp owns columns j (rows i)
    // 8 w .. 8 w + 7: ONE shared-memory load per k-step serves all products; coefficients come from the face records.
    constexpr int KS = 8;  // k-steps of a face stage (qf <= 32), RT = 2 row tiles of psi (pf = 16)
    const int pf = dv.pf, nfl = dv.n_lfe * pf;
    double psr[2][KS];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int gc = 4 * ks + tig, b = 8 * t + grp;
            psr[t][ks] = (gc < qf && b < pf) ? __ldg(dv.psi + b + pf * gc) : 0.0;
        }
    for (int lf = 0; lf < dv.n_lfe; ++lf, ++it) {
        produce();
        mbar_wait(full + slot, par);
        const double* St = ring + slot * stage_d + rowoff;
        const FaceRec<1, D>* fr = frec + lf * qf;
        const bool jw = warp == lf;  // J of this face: one warp
        double hg[1 + D][2][2], fa[2][2], ja[2][2][2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
#pragma unroll
            for (int w = 0; w <= D; ++w) hg[w][t][0] = hg[w][t][1] = 0.0;
            fa[t][0] = fa[t][1] = 0.0;
            ja[t][0][0] = ja[t][0][1] = ja[t][1][0] = ja[t][1][1] = 0.0;
        }
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            if (ks >= hks) break;
            const int gc = 4 * ks + tig;
            const bool live = gc < qf;
            const FaceRec<1, D>& r = fr[live ? gc : qf - 1];
            const double wg = live ? r.w : 0.0;
            const double ph = St[gc * kEsLd];
#pragma unroll
            for (int w = 0; w <= D; ++w) {
                const double b = (wg * (w == 0 ? r.dv_u[0] : r.dv_q[w - 1])) * ph;
#pragma unroll
                for (int t = 0; t < 2; ++t) dmma_8x8x4(hg[w][t][0], hg[w][t][1], psr[t][ks], b);
            }
            const double cf = wg * r.dfh_uh[0];
#pragma unroll
            for (int t = 0; t < 2; ++t) dmma_8x8x4(fa[t][0], fa[t][1], ph, psr[t][ks] * cf);
            if (jw) {
                const double cj = wg * r.dv_uh[0];
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int c = 0; c < 2; ++c) dmma_8x8x4(ja[t][c][0], ja[t][c][1], psr[t][ks], psr[c][ks] * cj);
            }
        }
            ring_release_all(empty + slot);
            if (++slot == kEsStages) { slot = 0; par ^= 1; }
        // ---- this face's blocks ----
        const int j0 = 8 * warp + 2 * tig;
#pragma unroll
        for (int w = 0; w <= D; ++w) {
            double* dst = (w == 0 ? out.H : out.G[w - 1]) + static_cast<size_t>(e) * nfl * kEsPe + lf * pf + grp;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(j0 + h) * nfl + 8 * t] = hg[w][t][h];
        }
        {
            double* dst = out.F + static_cast<size_t>(e) * kEsPe * nfl + rowoff;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(lf * pf + 8 * t + 2 * tig + h) * kEsPe] = fa[t][h];
        }
        if (jw) {
            double* dst = out.J + static_cast<size_t>(e) * nfl * nfl + lf * pf + grp;
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int c = 0; c < 2; ++c)
#pragma unroll
                    for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(lf * pf + 8 * c + 2 * tig + h) * nfl + 8 * t] = ja[t][c][h];
        }
    }
}

// ---- E and D_d of WIDE systems (M > 1, pe = 64: hex p = 3) through the same table ring ------------------------------
// One component pair (m, mp) per sweep of the point list, all 1 + D blocks of the pair resident (warp w: rows 8 w ..
// 8 w + 7 of four 64 x 64 blocks = 32 accumulator tiles; one CTA per SM, 255 registers).  The table ring keeps flowing
// across the M^2 sweeps.  The pair's coefficient rows -- 4 (1 + D) values per volume point, 1 + D per face point, scattered
// over the point records in the global (L2) scratch -- are gathered into a shared-memory table [point][18] by all
// threads, double-buffered: the loads of pair n + 1 are issued before the sweep of pair n and stored after it, so one
// CTA barrier per pair is the only synchronisation besides the ring's mbarriers.
constexpr int kEwLd = 18;  // coefficient row: 16 values + the weight + 1 (rows 144 bytes apart: 16-byte aligned, conflict-free 128-bit loads)
inline __host__ __device__ size_t ed_wide_doubles(int D, int qe, int nfp) {
    return ed_stream_doubles(D) + 2 * static_cast<size_t>(qe + nfp) * kEwLd;
}

template <int M, int D, int NW>
__device__ bool ed_stream_wide(const DiscView& dv, const LocalIn& in, const LocalOut& out, int e, const VolRec<M, D>* vrec,
                               const FaceRec<M, D>* frec, const int* s_orient, double* ring, uint64_t* bars, bool do_hgf) {
    static_assert(D == 3, "coefficient rows are laid out for 1 + D = 4 blocks");
    constexpr int NQ = 1 + D;
    constexpr int NH = NW / 8;           // column parts: 8 warps own all 64 columns of their rows, 16 warps half of them
    constexpr int NCT = kEsPe / 8 / NH;  // column tiles per warp
    constexpr int stage_d = (1 + D) * kEsPts * kEsLd;
    constexpr int NPAIR = M * M;
    constexpr int NCV = 4 * NQ + 1;  // table entries per volume point and pair: 4 (1 + D) coefficients + the quadrature weight
    constexpr int NCF = NQ + 1;      // per face point: 1 + D coefficients + the weight
    const int qe = dv.qe, qf = dv.qf, nfp = dv.n_lfe * qf, npe = M * kEsPe;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const int nsv = (qe + kEsPts - 1) / kEsPts, nsf = (nfp + kEsPts - 1) / kEsPts, nst = nsv + nsf;
    // after the M^2 sweeps: one ring stage per local face for H, G_d, F, J of all pairs (8-warp form only)
    constexpr int NCH = 6;                      // face coefficient sets per pair: dv_u, dv_q[0..2], dfh_uh, dv_uh (weight folded in)
    const int hks = (qf + 3) / 4;               // k-steps of a face stage
    const int pf = dv.pf, mpf = M * pf, nfl = dv.n_lfe * mpf;
    const int nith = 4 * hks * NPAIR * NCH;     // entries of a face's coefficient table [point][pair][set]
    const bool hgf = do_hgf && NW == 8 && pf == 16 && qf <= 32 && 2 * nith <= 2 * (qe + nfp) * kEwLd;
    const int n_ed = NPAIR * nst;
    const int total = n_ed + (hgf ? dv.n_lfe : 0);
    const int npt = qe + nfp;
    uint64_t* full = bars;
    uint64_t* empty = bars + kEsStages;
    const double dtv = in.dt_inv > 0.0 ? in.dt_inv : 0.0;
    double* cb = ring + kEsStages * stage_d;  // [2][npt][kEwLd]

    auto issue = [&](int gi, int slot) {
        if (lane != 0) return;
        double* dst = ring + slot * stage_d;
        if (gi >= n_ed) {  // face stage: all points of local face gi - n_ed
            const int lf = gi - n_ed;
            const uint32_t bytes = 4 * hks * kEsLd * sizeof(double);
            mbar_expect_tx(full + slot, bytes);
            tma_bulk_g2s(dst, dv.es_face + (static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf * kEsLd, bytes, full + slot);
            return;
        }
        const int s = gi % nst;
        if (s < nsv) {
            mbar_expect_tx(full + slot, stage_d * sizeof(double));
            tma_bulk_g2s(dst, dv.es_vol + static_cast<size_t>(s) * stage_d, stage_d * sizeof(double), full + slot);
        } else {
            constexpr uint32_t rb = kEsLd * sizeof(double);
            mbar_expect_tx(full + slot, kEsPts * rb);
            const int p0 = (s - nsv) * kEsPts;
            int p = p0;
            while (p < p0 + kEsPts) {
                const int pc = min(p, nfp - 1);
                const int lf = pc / qf, gc = pc - lf * qf;
                const int run = p < nfp ? min(min(p0 + kEsPts, nfp), (lf + 1) * qf) - p : 1;
                const double* src = dv.es_face + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * kEsLd;
                tma_bulk_g2s(dst + (p - p0) * kEsLd, src, run * rb, full + slot);
                p += run;
            }
        }
    };
    // coefficient gather of pair pr: this thread's items (item = (point, coefficient index)); loads first, stores later
    constexpr int kItems = 12 / NH;  // (8 warps) ceil((125 * 17 + 150 * 5) / 256) for the default rule; more points: extra trips
    const int nitem = qe * NCV + nfp * NCF;
    auto coef_ptr = [&](int pr, int item) -> const double* {
        const int mp = pr / M, m = pr - mp * M, mm = m * M + mp;
        if (item < qe * NCV) {
            const int pt = item / NCV, c = item - pt * NCV, w = c >> 2, k = c & 3;
            const VolRec<M, D>& r = vrec[pt];
            if (c == NCV - 1) return &r.w;
            if (w == 0) return k == 0 ? &r.dSu[mm] : &r.cE[mm * D + k - 1];
            return k == 0 ? &r.dSq[mm * D + w - 1] : &r.cD[((w - 1) * M * M + mm) * D + k - 1];
        }
        const int f = item - qe * NCV, pt = f / NCF, w = f - pt * NCF;
        const FaceRec<M, D>& r = frec[pt];
        if (w == NQ) return &r.w;
        return w == 0 ? &r.tau : &r.dfh_q[mm * D + w - 1];
    };
    auto coef_slot = [&](int item) -> int {
        if (item < qe * NCV) { const int pt = item / NCV; return pt * kEwLd + (item - pt * NCV); }
        const int f = item - qe * NCV, pt = f / NCF;
        return (qe + pt) * kEwLd + (f - pt * NCF);
    };
    auto gather_direct = [&](int pr, double* dstb) {  // first pair, and the tail items beyond kItems trips
        for (int item = tid; item < nitem; item += nt) dstb[coef_slot(item)] = __ldcg(coef_ptr(pr, item));
    };

    __syncthreads();  // earlier users of this shared memory (generic proxy) are done
    if (warp == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int it = 0; it < kEsStages - 1 && it < total; ++it) issue(it, it);
    }
    gather_direct(0, cb);
    __syncthreads();

    const int rowoff = 8 * (warp & 7) + grp;
    const int col0 = (warp >> 3) * NCT * 8;  // first column of this warp's tiles
    int slot = 0, par = 0, it = 0;
    auto produce = [&]() {
        if (warp != 0) return;
        const int nx = it + kEsStages - 1;
        if (nx < total) {
            int nslot = slot + kEsStages - 1;
            if (nslot >= kEsStages) nslot -= kEsStages;
            if (it >= 1) mbar_wait(empty + nslot, ((it - 1) / kEsStages) & 1);
            issue(nx, nslot);
        }
    };
    for (int pr = 0; pr < NPAIR; ++pr) {
        const int mp = pr / M, m = pr - mp * M;
        const double* cbp = cb + static_cast<size_t>(pr & 1) * npt * kEwLd;
        double* cbn = cb + static_cast<size_t>((pr + 1) & 1) * npt * kEwLd;
        const double dte = (m == mp) ? dtv : 0.0;
        // next pair's coefficients: loads in flight during this pair's sweep
        double cst[kItems];
        const bool more = pr + 1 < NPAIR;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const int item = tid + j * nt;
            cst[j] = (more && item < nitem) ? __ldcg(coef_ptr(pr + 1, item)) : 0.0;
        }
        double acc[NQ][NCT][2];
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
            for (int b = 0; b < NCT; ++b) acc[q][b][0] = acc[q][b][1] = 0.0;
        for (int s = 0; s < nst; ++s, ++it) {
            produce();
            mbar_wait(full + slot, par);
            const double* St = ring + slot * stage_d;
            const bool vol = s < nsv;
            const int p0 = vol ? s * kEsPts : (s - nsv) * kEsPts;
            const int npts = vol ? qe : nfp;
            // left fragments of both k-steps first (their loads and FMA chains overlap), then the products
            double a[kEsPts / 4][NQ];
#pragma unroll
            for (int ks = 0; ks < kEsPts / 4; ++ks) {
                const int p = 4 * ks + tig;
                const bool live = p0 + p < npts;
                const int pt = live ? p0 + p : npts - 1;
                if (vol) {
                    const double2* cr = reinterpret_cast<const double2*>(cbp + pt * kEwLd);
                    const double nw = live ? -cbp[pt * kEwLd + NCV - 1] : 0.0;
                    const double t0 = St[p * kEsLd + rowoff];
                    double tk[D];
#pragma unroll
                    for (int k = 0; k < D; ++k) tk[k] = St[((1 + k) * kEsPts + p) * kEsLd + rowoff];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        const double2 c01 = cr[2 * q], c23 = cr[2 * q + 1];
                        double v = (q == 0 ? c01.x - dte : c01.x) * t0;
                        v = fma(c01.y, tk[0], v);
                        v = fma(c23.x, tk[1], v);
                        v = fma(c23.y, tk[2], v);
                        a[ks][q] = nw * v;
                    }
                } else {
                    const double2* cr = reinterpret_cast<const double2*>(cbp + (qe + pt) * kEwLd);
                    const double wq = live ? cbp[(qe + pt) * kEwLd + NQ] : 0.0;
                    const double t0 = wq * St[p * kEsLd + rowoff];
                    const double2 c01 = cr[0], c23 = cr[1];
                    a[ks][0] = (m == mp ? c01.x : 0.0) * t0;
                    a[ks][1] = c01.y * t0;
                    a[ks][2] = c23.x * t0;
                    a[ks][3] = c23.y * t0;
                }
            }
#pragma unroll
            for (int ks = 0; ks < kEsPts / 4; ++ks) {
                const double* bs = St + (4 * ks + tig) * kEsLd + col0 + grp;
#pragma unroll
                for (int b = 0; b < NCT; ++b) {
                    const double bf = bs[8 * b];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) dmma_8x8x4(acc[q][b][0], acc[q][b][1], a[ks][q], bf);
                }
            }
            ring_release_all(empty + slot);
            if (++slot == kEsStages) { slot = 0; par ^= 1; }
        }
        // ---- this pair's blocks: rows (m, i), columns (mp, j) ----
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double* dst = (q == 0 ? out.E : out.Dm[q - 1]) + static_cast<size_t>(e) * npe * npe +
                          static_cast<size_t>(mp * kEsPe) * npe + m * kEsPe + rowoff;
#pragma unroll
            for (int b = 0; b < NCT; ++b)
#pragma unroll
                for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(col0 + 8 * b + 2 * tig + h) * npe] = acc[q][b][h];
        }
        // next pair's coefficient table (the other buffer: its last readers passed the previous barrier)
        if (more) {
#pragma unroll
            for (int j = 0; j < kItems; ++j) {
                const int item = tid + j * nt;
                if (item < nitem) cbn[coef_slot(item)] = cst[j];
            }
            for (int item = tid + kItems * nt; item < nitem; item += nt) cbn[coef_slot(item)] = __ldcg(coef_ptr(pr + 1, item));
        }
        __syncthreads();
    }
    if (!hgf) return false;
    // ---- H, G_d, F, J of all component pairs, one ring stage per local face ----
    // [H | G_d](lf m b, mp j) = sum_gc psi_b(gc) (cw(gc) phis_j(gc)),  F(m i, lf mp bp) = sum_gc phis_i(gc) (cf(gc) psi_bp(gc)),
    // J(lf m b, lf mp bp) = sum_gc psi_b(gc) (cj(gc) psi_bp(gc)).  psi lives in registers (left fragment of H / G_d / J, right
    // fragment of F / J), the face's trace-table fragments are read once from the ring and serve all M^2 pairs, the pairs'
    // weighted coefficients come from a shared-memory table gathered per face from the record scratch (double-buffered).
    constexpr int KS = 8;
    constexpr int kItemsH = 17;  // ceil(28 * 25 * 6 / 256) for M = 5 and the default rule; more: extra trips
    double* hb = cb;             // [2][nith]
    auto hcoef = [&](int lf, int item) -> double {
        const int gc = item / (NPAIR * NCH), rem = item - gc * (NPAIR * NCH);
        const int pr = rem / NCH, c = rem - pr * NCH;
        if (gc >= qf) return 0.0;
        const int mp = pr / M, m = pr - mp * M, mm = m * M + mp;
        const FaceRec<M, D>& r = frec[lf * qf + gc];
        const double* v = c == 0 ? &r.dv_u[mm] : (c <= D ? &r.dv_q[mm * D + c - 1] : (c == 1 + D ? &r.dfh_uh[mm] : &r.dv_uh[mm]));
        return __ldcg(&r.w) * __ldcg(v);
    };
    for (int item = tid; item < nith; item += nt) hb[item] = hcoef(0, item);
    double psr[2][KS];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
            const int gc = 4 * ks + tig, bb = 8 * t + grp;
            psr[t][ks] = (gc < qf && bb < pf) ? __ldg(dv.psi + bb + pf * gc) : 0.0;
        }
    __syncthreads();
    for (int lf = 0; lf < dv.n_lfe; ++lf, ++it) {
        const double* hbp = hb + static_cast<size_t>(lf & 1) * nith;
        double* hbn = hb + static_cast<size_t>((lf + 1) & 1) * nith;
        const bool more = lf + 1 < dv.n_lfe;
        double hst[kItemsH];
#pragma unroll
        for (int j = 0; j < kItemsH; ++j) {
            const int item = tid + j * nt;
            hst[j] = (more && item < nith) ? hcoef(lf + 1, item) : 0.0;
        }
        produce();
        mbar_wait(full + slot, par);
        const double* St = ring + slot * stage_d + rowoff;
        double ph[KS];
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) ph[ks] = ks < hks ? St[(4 * ks + tig) * kEsLd] : 0.0;
        ring_release_all(empty + slot);  // the fragments are in registers
        if (++slot == kEsStages) { slot = 0; par ^= 1; }
        const int j0 = 8 * warp + 2 * tig;
        for (int pr = 0; pr < NPAIR; ++pr) {
            const int mp = pr / M, m = pr - mp * M;
            const bool jw = (pr & 7) == warp;  // J block of this (face, pair): one warp
            double hg[1 + D][2][2], fa[2][2], ja[2][2][2];
#pragma unroll
            for (int t = 0; t < 2; ++t) {
#pragma unroll
                for (int w = 0; w <= D; ++w) hg[w][t][0] = hg[w][t][1] = 0.0;
                fa[t][0] = fa[t][1] = 0.0;
                ja[t][0][0] = ja[t][0][1] = ja[t][1][0] = ja[t][1][1] = 0.0;
            }
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                if (ks >= hks) break;
                const double2* cr = reinterpret_cast<const double2*>(hbp + (static_cast<size_t>(4 * ks + tig) * NPAIR + pr) * NCH);
                const double2 c01 = cr[0], c23 = cr[1], c45 = cr[2];
                const double cwv[1 + D] = {c01.x, c01.y, c23.x, c23.y};
#pragma unroll
                for (int w = 0; w <= D; ++w) {
                    const double bq = cwv[w] * ph[ks];
#pragma unroll
                    for (int t = 0; t < 2; ++t) dmma_8x8x4(hg[w][t][0], hg[w][t][1], psr[t][ks], bq);
                }
#pragma unroll
                for (int t = 0; t < 2; ++t) dmma_8x8x4(fa[t][0], fa[t][1], ph[ks], psr[t][ks] * c45.x);
                if (jw) {
#pragma unroll
                    for (int t = 0; t < 2; ++t)
#pragma unroll
                        for (int c = 0; c < 2; ++c) dmma_8x8x4(ja[t][c][0], ja[t][c][1], psr[t][ks], psr[c][ks] * c45.y);
                }
            }
#pragma unroll
            for (int w = 0; w <= D; ++w) {
                double* dst = (w == 0 ? out.H : out.G[w - 1]) + static_cast<size_t>(e) * nfl * npe +
                              static_cast<size_t>(mp * kEsPe + j0) * nfl + lf * mpf + m * pf + grp;
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(h) * nfl + 8 * t] = hg[w][t][h];
            }
            {
                double* dst = out.F + static_cast<size_t>(e) * npe * nfl + static_cast<size_t>(lf * mpf + mp * pf) * npe + m * kEsPe + rowoff;
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(8 * t + 2 * tig + h) * npe] = fa[t][h];
            }
            if (jw) {
                double* dst = out.J + static_cast<size_t>(e) * nfl * nfl + static_cast<size_t>(lf * mpf + mp * pf) * nfl + lf * mpf + m * pf + grp;
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int c = 0; c < 2; ++c)
#pragma unroll
                        for (int h = 0; h < 2; ++h) dst[static_cast<size_t>(8 * c + 2 * tig + h) * nfl + 8 * t] = ja[t][c][h];
            }
        }
        if (more) {
#pragma unroll
            for (int j = 0; j < kItemsH; ++j) {
                const int item = tid + j * nt;
                if (item < nith) hbn[item] = hst[j];
            }
            for (int item = tid + kItemsH * nt; item < nith; item += nt) hbn[item] = hcoef(lf + 1, item);
        }
        __syncthreads();
    }
    return true;
}

// ---- H, G_d and F of scalar systems (M = 1) on the tensor-core path ------------------------------------------
// Per local face lf (K = the qf face points):
//   [H | G_0 .. G_{D-1}](lf b, j) = sum_gc psi_b(gc) * (c_w(gc) w_gc phis_j(gc)),  c_0 = dv_u, c_{1+dp} = dv_q[dp]
//   F(i, lf bp)                   = sum_gc phis_i(gc) * (w_gc dfh_uh(gc) psi_bp(gc))
// (local_ops.cpp:186-219).  psi^T and phis are the left operands, the coefficient-scaled tables the right ones.
constexpr int kHgfRtMax = 4;  // 8-row tiles covering pf (pf <= 32)
// The per-point coefficients are applied to the operand FRAGMENTS: with cw(gc) = w_gc c(gc),
//   [H | G_dp](lf b, j) = sum_gc psi_b(gc) * (cw(gc) phis_j(gc)),     F(i, lf bp) = sum_gc phis_i(gc) * (cf(gc) psi_bp(gc)),
// so per local face only the trace table phis (qf x pe) and a small table of coefficients -- M^2 (2 + D) values per
// face point, ALL component pairs at once -- are staged; psi^T is staged once per element.  A warp owns an 8-column
// tile of j (resp. an 8-row tile of i), keeps its phis fragments in registers and walks all (component pair,
// coefficient set) units of the face scaling the fragment by cw on the fly: two barriers per face, none per pair.
// Operands are k-major ([face point][row or column], leading dimensions = 4 mod 16): conflict-free DMMA fragment loads.
constexpr int kHgfKsMax = 10;  // k-steps of 4 face points (qf <= 40)
struct HgfPlan {
    int pfp, qfp, ldp, lda, pep;
    __host__ __device__ size_t doubles(int D, int M) const {
        return static_cast<size_t>(qfp) * ldp + static_cast<size_t>(qfp) * lda + static_cast<size_t>(M) * M * (2 + D) * qfp;
    }
};
inline __host__ __device__ HgfPlan hgf_plan(int pe, int pf, int qf) {
    HgfPlan p;
    p.pfp = (pf + 7) / 8 * 8;
    p.pep = (pe + 7) / 8 * 8;
    p.qfp = (qf + 3) / 4 * 4;
    p.ldp = (p.pfp + 15) / 16 * 16 + 4;
    p.lda = (p.pep + 15) / 16 * 16 + 4;
    return p;
}
inline bool hgf_dmma_ok(int pf, int qf) { return pf <= 8 * kHgfRtMax && qf <= 4 * kHgfKsMax; }

template <int M, int D, bool GREC>
__device__ void hgf_dmma(const DiscView& dv, const LocalOut& out, int e, const FaceRec<M, D>* frec, const int* s_orient,
                         double* buf) {
    // Rows / columns of component pair (m, mp) inside the blocks: H, G (nfl x npe): row lf mpf + m pf + b, column
    // mp pe + j;  F (npe x nfl): row m pe + i, column lf mpf + mp pf + bp.  Coefficient sets of a pair: 0 = dv_u (H),
    // 1 + dp = dv_q[dp] (G_dp), 1 + D = dfh_uh (F).
    constexpr int NC = 2 + D;
    const int pe = dv.pe, pf = dv.pf, qf = dv.qf, n_lfe = dv.n_lfe;
    const int mpf = M * pf, nfl = n_lfe * mpf, npe = M * pe;
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarps = nt >> 5;
    const int grp = lane >> 2, tig = lane & 3;
    const HgfPlan pl = hgf_plan(pe, pf, qf);
    const int ldp = pl.ldp, lda = pl.lda, qfp = pl.qfp;
    double* Ps = buf;               // psi^T:         [gc][b]
    double* Fs = Ps + qfp * ldp;    // phis:          [gc][i]
    double* Cw = Fs + qfp * lda;    // coefficients:  [pair][set][gc]
    __syncthreads();
    for (int t = tid; t < static_cast<int>(pl.doubles(D, M)); t += nt) buf[t] = 0.0;
    __syncthreads();
    for (int t = tid; t < qf * pf; t += nt) {
        const int gc = t / pf, b = t - gc * pf;
        Ps[gc * ldp + b] = __ldg(dv.psi + b + pf * gc);
    }
    const int rt_h = pl.pfp / 8, ct_h = pl.pep / 8;  // 8-row tiles over b / bp, 8-column tiles over j (= row tiles over i)
    const int ksteps = qfp / 4;
    const int hw = tid >> 4, l16 = tid & 15, nhw = nt >> 4;  // staging: half-warp <-> face point, lanes <-> basis function
    for (int lf = 0; lf < n_lfe; ++lf) {
        const double* tp = dv.tphi + (static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf * pe;
        const FaceRec<M, D>* fr = frec + lf * qf;
        __syncthreads();  // the previous face's tiles are done with Fs, Cw
        for (int gc = hw; gc < qf; gc += nhw)
            for (int j = l16; j < pe; j += 16) Fs[gc * lda + j] = __ldg(tp + static_cast<size_t>(gc) * pe + j);
        for (int t = tid; t < M * M * qf; t += nt) {
            const int pr = t / qf, gc = t - pr * qf;
            const int mp = pr / M, m = pr - mp * M, mm = m * M + mp;
            const FaceRec<M, D>& r = fr[gc];
            const double wg = rec_ld<GREC>(&r.w);
            double* cw = Cw + pr * NC * qfp + gc;
            cw[0] = wg * rec_ld<GREC>(&r.dv_u[mm]);
#pragma unroll
            for (int dq = 0; dq < D; ++dq) cw[(1 + dq) * qfp] = wg * rec_ld<GREC>(&r.dv_q[mm * D + dq]);
            cw[(1 + D) * qfp] = wg * rec_ld<GREC>(&r.dfh_uh[mm]);
        }
        __syncthreads();
        // ---- H / G_d: this warp's column tiles of j ----
        for (int ct = warp; ct < ct_h; ct += nwarps) {
            double bf[kHgfKsMax];
#pragma unroll
            for (int ks = 0; ks < kHgfKsMax; ++ks) bf[ks] = ks < ksteps ? Fs[(4 * ks + tig) * lda + ct * 8 + grp] : 0.0;
            const int j = ct * 8 + 2 * tig;
            for (int pr = 0; pr < M * M; ++pr) {
                const int mp = pr / M, m = pr - mp * M;
                for (int w = 0; w <= D; ++w) {
                    const double* cw = Cw + (pr * NC + w) * qfp + tig;
                    double c[kHgfRtMax][2];
#pragma unroll
                    for (int rt = 0; rt < kHgfRtMax; ++rt) c[rt][0] = c[rt][1] = 0.0;
#pragma unroll
                    for (int ks = 0; ks < kHgfKsMax; ++ks) {
                        if (ks >= ksteps) break;
                        const double b = bf[ks] * cw[4 * ks];
                        const double* as = Ps + (4 * ks + tig) * ldp + grp;
#pragma unroll
                        for (int rt = 0; rt < kHgfRtMax; ++rt)
                            if (rt < rt_h) dmma_8x8x4(c[rt][0], c[rt][1], as[rt * 8], b);
                    }
                    double* dst = (w == 0 ? out.H : out.G[w - 1]) + static_cast<size_t>(e) * nfl * npe;
#pragma unroll
                    for (int rt = 0; rt < kHgfRtMax; ++rt) {
                        const int bb = rt * 8 + grp;
                        if (rt >= rt_h || bb >= pf) continue;
                        const size_t row = lf * mpf + m * pf + bb;
                        if (j < pe) dst[static_cast<size_t>(mp * pe + j) * nfl + row] = c[rt][0];
                        if (j + 1 < pe) dst[static_cast<size_t>(mp * pe + j + 1) * nfl + row] = c[rt][1];
                    }
                }
            }
        }
        // ---- F (rows i, columns bp): this warp's row tiles of i ----
        for (int rti = warp; rti < ct_h; rti += nwarps) {
            double af[kHgfKsMax];
#pragma unroll
            for (int ks = 0; ks < kHgfKsMax; ++ks) af[ks] = ks < ksteps ? Fs[(4 * ks + tig) * lda + rti * 8 + grp] : 0.0;
            const int i = rti * 8 + grp;
            double* dst = out.F + static_cast<size_t>(e) * npe * nfl;
            for (int pr = 0; pr < M * M; ++pr) {
                const int mp = pr / M, m = pr - mp * M;
                const double* cf = Cw + (pr * NC + 1 + D) * qfp + tig;
                double c[kHgfRtMax][2];
#pragma unroll
                for (int cb = 0; cb < kHgfRtMax; ++cb) c[cb][0] = c[cb][1] = 0.0;
#pragma unroll
                for (int ks = 0; ks < kHgfKsMax; ++ks) {
                    if (ks >= ksteps) break;
                    const double cfk = cf[4 * ks];
                    const double* bs = Ps + (4 * ks + tig) * ldp + grp;
#pragma unroll
                    for (int cb = 0; cb < kHgfRtMax; ++cb)
                        if (cb < rt_h) dmma_8x8x4(c[cb][0], c[cb][1], af[ks], bs[cb * 8] * cfk);
                }
                const size_t row = m * pe + i;
#pragma unroll
                for (int cb = 0; cb < kHgfRtMax; ++cb) {
                    const int bp = cb * 8 + 2 * tig;
                    if (cb >= rt_h || i >= pe) continue;
                    if (bp < pf) dst[static_cast<size_t>(lf * mpf + mp * pf + bp) * npe + row] = c[cb][0];
                    if (bp + 1 < pf) dst[static_cast<size_t>(lf * mpf + mp * pf + bp + 1) * npe + row] = c[cb][1];
                }
            }
        }
    }
}

// RES: residual-only specialisation (assemble_residual: once per Newton step and per line-search trial).  Without the
// Jacobian code the kernel needs half the registers, so four CTAs per SM cover each other's load latency.
template <class Model, int NT, bool ED, bool GREC, bool RES = false>
__global__ void __launch_bounds__(NT, RES ? (Model::M == 1 ? 4 : 2) : ((!GREC && Model::M == 1 && NT <= 256) ? 2 : 1)) local_assemble_kernel(DiscView dv, ModelView mv, LocalIn in, LocalOut out,
                                                            int want_jac, int gv0, int gv1, int fp0, int fp1, int first,
                                                            int ed_dmma_on, char* rec_scratch, size_t rec_stride) {
    // GREC: the point records of wide systems do not fit shared memory; they are staged per element in a
    // global scratch buffer (written and re-read by the same CTA, i.e. served from L2), which keeps the
    // whole point sweep in ONE launch and leaves shared memory to the tensor-core operand tiles.
    // Point records of the volume points [gv0, gv1) and face points [fp0, fp1) live in shared memory.
    // When all points of an element fit (scalar models) there is ONE launch (first = 1) and every
    // output entry is written once.  Wide systems (M = 5) are swept in several launches over point
    // chunks that accumulate into the outputs -- still volume points ascending, then faces.
    constexpr int M = Model::M, D = Model::D;
    using VR = VolRec<M, D>;
    using FR = FaceRec<M, D>;
    extern __shared__ double sm[];
    const int e = blockIdx.x;
    const int pe = dv.pe, pf = dv.pf, qe = dv.qe, qf = dv.qf, n_lfe = dv.n_lfe;
    const int npe = M * pe, mpf = M * pf, nfl = n_lfe * mpf;
    [[maybe_unused]] const int nfp = n_lfe * qf;
    const int tid = threadIdx.x, nt = blockDim.x;

    double* us = sm;                  // npe
    double* qs = us + npe;            // D*npe  (direction-major)
    double* uhs = qs + D * npe;       // nfl
    double* ups = uhs + nfl;          // npe
    double* red = ups + npe;          // kResParts * npe: partial residual sums
    VR* vrec;
    FR* frec;
    double* opbuf_base;
    if constexpr (GREC) {
        char* base = rec_scratch + static_cast<size_t>(blockIdx.x) * rec_stride;
        vrec = reinterpret_cast<VR*>(base);
        frec = reinterpret_cast<FR*>(vrec + (gv1 - gv0));
        opbuf_base = red + ((kResParts * npe + 1) & ~1);
    } else {
        vrec = reinterpret_cast<VR*>(red + kResParts * npe);
        frec = reinterpret_cast<FR*>(vrec + (gv1 - gv0));
        opbuf_base = sm + ((reinterpret_cast<const char*>(frec + (fp1 - fp0)) - reinterpret_cast<const char*>(sm) + 15) / 16) * 2;
    }
    __shared__ int s_face[8], s_side[8], s_orient[8], s_tag[8];
    __shared__ uint64_t s_bars[2 * kEsStages];  // full / empty mbarriers of ed_stream's table ring
    if constexpr (ED && D == 3 && ((NT == 256 && (M == 1) != GREC) || (NT == 512 && M > 1 && GREC))) {
        if (tid == 0) {
            for (int i = 0; i < kEsStages; ++i) {
                mbar_init(s_bars + i, 1);
                mbar_init(s_bars + kEsStages + i, NT);  // every thread releases a stage for itself (tma.cuh: ring_release_all)
            }
            mbar_fence_init();
        }
    }

    const Model model(mv);
    const bool transient = in.dt_inv > 0.0;

    for (int t = tid; t < npe; t += nt) {
        us[t] = in.u[static_cast<size_t>(e) * npe + t];
        for (int d = 0; d < D; ++d) qs[d * npe + t] = in.q[d][static_cast<size_t>(e) * npe + t];
        ups[t] = transient ? in.u_prev[static_cast<size_t>(e) * npe + t] : 0.0;
    }
    if (tid < n_lfe) {
        const int f = dv.elem_faces[e * n_lfe + tid];
        const int side = dv.elem_side[e * n_lfe + tid];
        s_face[tid] = f;
        s_side[tid] = side;
        s_orient[tid] = dv.face_orient[2 * f + side];
        s_tag[tid] = dv.bnd_tag[f];
    }
    for (int t = tid; t < nfl; t += nt) {
        const int lf = t / mpf;
        uhs[t] = in.uhat[static_cast<size_t>(dv.elem_faces[e * n_lfe + lf]) * mpf + (t - lf * mpf)];
    }
    __syncthreads();

    // ---- phase 1a: volume points ----
    for (int g = gv0 + tid; g < gv1; g += nt) {
        const size_t gi = static_cast<size_t>(e) * qe + g;
        VR& r = vrec[g - gv0];
        const double* phig = dv.phi + static_cast<size_t>(pe) * g;
        double ug[M], qg[M * D], upg[M];
        for (int m = 0; m < M; ++m) {
            double a = 0.0, ap = 0.0, aq[D];
            for (int d = 0; d < D; ++d) aq[d] = 0.0;
            for (int i = 0; i < pe; ++i) {
                const double p = phig[i];
                a += us[m * pe + i] * p;
                for (int d = 0; d < D; ++d) aq[d] += qs[d * npe + m * pe + i] * p;
                if (transient) ap += ups[m * pe + i] * p;
            }
            ug[m] = a;
            upg[m] = ap;
            for (int d = 0; d < D; ++d) qg[m * D + d] = aq[d];
        }
        r.w = dv.wq[g] * dv.elem_detjac[gi];
        const double* ij = dv.elem_invjac + gi * D * D;  // ij[r*D + d] = d xi_r / d x_d
        const double* x = dv.elem_coords + gi * D;
        const double* f = mv.forcing_q ? mv.forcing_q + gi * M : nullptr;
        double Fl[M * D];
        model.flux(ug, qg, x, Fl);
        model.source(ug, qg, x, f, r.S);
        for (int m = 0; m < M; ++m) {
            r.tm[m] = transient ? in.dt_inv * (ug[m] - upg[m]) : 0.0;
            for (int rr = 0; rr < D; ++rr) {
                double sfl = 0.0;
                for (int d = 0; d < D; ++d) sfl += Fl[m * D + d] * ij[rr * D + d];
                r.Fr[m * D + rr] = sfl;
            }
        }
        if (!RES && want_jac) {
            double dFu[M * D * M], dFq[M * D * M * D];
            model.dflux_du(ug, qg, x, dFu);
            model.dflux_dq(ug, qg, x, dFq);
            model.dsource_du(ug, qg, x, r.dSu);
            model.dsource_dq(ug, qg, x, r.dSq);
            for (int m = 0; m < M; ++m)
                for (int mp = 0; mp < M; ++mp)
                    for (int rr = 0; rr < D; ++rr) {
                        double se = 0.0;
                        for (int d = 0; d < D; ++d) se += dFu[(m * D + d) * M + mp] * ij[rr * D + d];
                        r.cE[(m * M + mp) * D + rr] = se;
                        for (int dp = 0; dp < D; ++dp) {
                            double sd = 0.0;
                            for (int d = 0; d < D; ++d) sd += dFq[((m * D + d) * M + mp) * D + dp] * ij[rr * D + d];
                            r.cD[((dp * M + m) * M + mp) * D + rr] = sd;
                        }
                    }
        }
    }
    // ---- phase 1b: face points ----
    for (int p = fp0 + tid; p < fp1; p += nt) {
        const int lf = p / qf, gc = p - lf * qf;
        const int f = s_face[lf], side = s_side[lf], tag = s_tag[lf];
        FR& r = frec[p - fp0];
        const size_t fi = static_cast<size_t>(f) * qf + gc;
        const double* phis = dv.tphi + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe;
        const double* psic = dv.psi + static_cast<size_t>(pf) * gc;
        const double* n = dv.face_normal + ((static_cast<size_t>(f) * 2 + side) * qf + gc) * D;
        const double* x = dv.face_coords + fi * D;
        double ug[M], qg[M * D], uh[M];
        for (int m = 0; m < M; ++m) {
            double a = 0.0, aq[D];
            for (int d = 0; d < D; ++d) aq[d] = 0.0;
            for (int i = 0; i < pe; ++i) {
                const double ph = phis[i];
                a += us[m * pe + i] * ph;
                for (int d = 0; d < D; ++d) aq[d] += qs[d * npe + m * pe + i] * ph;
            }
            ug[m] = a;
            for (int d = 0; d < D; ++d) qg[m * D + d] = aq[d];
            double h = 0.0;
            for (int b = 0; b < pf; ++b) h += uhs[lf * mpf + m * pf + b] * psic[b];
            uh[m] = h;
        }
        r.w = dv.wf[gc] * dv.face_detjac[fi];
        const double tau = model.tau_fn(ug, uh, n);
        r.tau = tau;
        double Fl[M * D];
        model.flux(uh, qg, x, Fl);
        for (int m = 0; m < M; ++m) {
            double fn = 0.0;
            for (int d = 0; d < D; ++d) fn += Fl[m * D + d] * n[d];
            r.fhat[m] = fn + tau * (ug[m] - uh[m]);
        }
        if constexpr (RES) {
            // residual only: the face contribution needs fhat (interior faces) or the boundary value, no derivatives
            if (tag == 0) {
                for (int m = 0; m < M; ++m) r.val[m] = r.fhat[m];
            } else {
                BFlux<M, D> b;
                const double* gD = mv.dirichlet_q ? mv.dirichlet_q + fi * M : nullptr;
                model.boundary(tag, ug, qg, uh, n, x, gD, b);
                for (int m = 0; m < M; ++m) r.val[m] = b.val[m];
            }
        } else {
            double dFu[M * D * M], dFq[M * D * M * D];
            if (want_jac || tag != 0) {
                model.dflux_du(uh, qg, x, dFu);
                model.dflux_dq(uh, qg, x, dFq);
            } else {
                for (int k = 0; k < M * D * M; ++k) dFu[k] = 0.0;
                for (int k = 0; k < M * D * M * D; ++k) dFq[k] = 0.0;
            }
            // derivatives of the numerical flux (local_ops.cpp:186-189)
            for (int m = 0; m < M; ++m)
                for (int mp = 0; mp < M; ++mp) {
                    double su = 0.0;
                    for (int d = 0; d < D; ++d) su += dFu[(m * D + d) * M + mp] * n[d];
                    r.dfh_uh[m * M + mp] = su - ((m == mp) ? tau : 0.0);
                    for (int dp = 0; dp < D; ++dp) {
                        double sq = 0.0;
                        for (int d = 0; d < D; ++d) sq += dFq[((m * D + d) * M + mp) * D + dp] * n[d];
                        r.dfh_q[(m * M + mp) * D + dp] = sq;
                    }
                }
            if (tag == 0) {
                for (int m = 0; m < M; ++m) r.val[m] = r.fhat[m];
                for (int k = 0; k < M * M; ++k) {
                    r.dv_u[k] = ((k / M) == (k % M)) ? tau : 0.0;
                    r.dv_uh[k] = r.dfh_uh[k];
                }
                for (int k = 0; k < M * M * D; ++k) r.dv_q[k] = r.dfh_q[k];
            } else {
                BFlux<M, D> b;
                const double* gD = mv.dirichlet_q ? mv.dirichlet_q + fi * M : nullptr;
                model.boundary(tag, ug, qg, uh, n, x, gD, b);
                for (int m = 0; m < M; ++m) r.val[m] = b.val[m];
                for (int k = 0; k < M * M; ++k) { r.dv_u[k] = b.d_u[k]; r.dv_uh[k] = b.d_uh[k]; }
                for (int k = 0; k < M * M * D; ++k) r.dv_q[k] = b.d_q[k];
            }
        }
    }
    __syncthreads();

    // ---- phase 2a: residuals (negated weak residuals, local_ops.cpp:223-226).  The point sweep of basis
    // function i is split over NP thread groups (contiguous point ranges, volume points first); the partial
    // sums are combined in ascending range order, so the result does not depend on timing ----
    {
        const int NP = min(kResParts, max(1, nt / pe));
        const int nvp = gv1 - gv0, ntot = nvp + (fp1 - fp0);
        for (int t = tid; t < NP * pe; t += nt) {  // one trip unless pe > nt (then NP = 1)
            const int part = t / pe, i = t - part * pe;
            const int q0 = static_cast<int>(static_cast<long long>(ntot) * part / NP);
            const int q1 = static_cast<int>(static_cast<long long>(ntot) * (part + 1) / NP);
            double acc[M];
            for (int m = 0; m < M; ++m) acc[m] = 0.0;
            for (int q = q0; q < min(q1, nvp); ++q) {
                const int g = gv0 + q;
                const VR& r = vrec[q];
                const double ph = dv.phi[i + pe * g];
                double dp_[D];
                for (int k = 0; k < D; ++k) dp_[k] = dv.dphi[k][i + pe * g];
                for (int m = 0; m < M; ++m) {
                    double fg = 0.0;
                    for (int k = 0; k < D; ++k) fg += r.Fr[m * D + k] * dp_[k];
                    double v = -fg - r.S[m] * ph;
                    if (transient) v += r.tm[m] * ph;
                    acc[m] += r.w * v;
                }
            }
            for (int q = max(q0, nvp); q < q1; ++q) {
                const int p = fp0 + q - nvp;
                const int lf = p / qf, gc = p - lf * qf;
                const FR& r = frec[p - fp0];
                const double ph = dv.tphi[((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe + i];
                for (int m = 0; m < M; ++m) acc[m] += r.w * r.fhat[m] * ph;
            }
            for (int m = 0; m < M; ++m) red[(part * M + m) * pe + i] = acc[m];
        }
        __syncthreads();
        for (int t = tid; t < npe; t += nt) {
            const int m = t / pe, i = t - m * pe;
            double a = 0.0;
            for (int part = 0; part < NP; ++part) a += red[(part * M + m) * pe + i];
            double* o = out.ru + static_cast<size_t>(e) * npe + t;
            *o = first ? -a : *o - a;
        }
    }
    for (int t = tid; t < n_lfe * pf; t += nt) {
        const int lf = t / pf, b = t - lf * pf;
        double acc[M];
        for (int m = 0; m < M; ++m) acc[m] = 0.0;
        const int g0 = max(0, fp0 - lf * qf), g1 = min(qf, fp1 - lf * qf);
        for (int gc = g0; gc < g1; ++gc) {
            const FR& r = frec[lf * qf + gc - fp0];
            const double ps = dv.psi[b + pf * gc];
            for (int m = 0; m < M; ++m) acc[m] += r.w * r.val[m] * ps;
        }
        for (int m = 0; m < M; ++m) {
            double* o = out.ruhat_e + static_cast<size_t>(e) * nfl + lf * mpf + m * pf + b;
            *o = first ? -acc[m] : *o - acc[m];
        }
    }
    if (RES || !want_jac) return;

    // ---- phase 2b: E and D_d.  A thread owns a TI x TJ tile of scalar-basis pairs (i, j); per point it
    // forms the i-side values once and rank-1 updates the tile.  Component columns mp are swept one
    // at a time so that the accumulators (M (1 + D) per pair) stay in registers for wide systems ----
    int dbg_skip = (ed_dmma_on >> 4) & 7;  // measurement aid (hdgb_set_tuning "local_debug_skip"): 1 = E/D_d, 2 = H/G_d/F
    // launcher: pe = 64 scalar system, all points in this launch; bit 3: E / D_d streamed, bit 7: H / G_d / F / J streamed
    const bool ed_streamed = ed_dmma_on & 8, hgf_streamed = ed_dmma_on & 128, split_copies = ed_dmma_on & 256;
    ed_dmma_on &= 7;
    bool hgf_done = false, j_done = false;
    if constexpr (ED && M == 1 && D == 3 && !GREC && NT == 256) {
        if (ed_streamed || hgf_streamed) {
            // table ring + fragment-built operands: E, D_d, then H, G_d, F, J -- one barrier-free pipeline.  J's entries
            // outside the per-face diagonal blocks are zero.
            const bool hs = hgf_streamed && ed_dmma_on == 2 && pf == 16 && qf <= 32 && 4 * ((qf + 3) / 4) <= (1 + D) * kEsPts;
            if (hs && !(dbg_skip & 2)) {
                for (int t = tid; t < nfl * nfl; t += nt) {
                    const int c = t / nfl, r = t - c * nfl;
                    if (c / pf != r / pf) out.J[static_cast<size_t>(e) * nfl * nfl + t] = 0.0;
                }
            }
            if (!ed_streamed && !(dbg_skip & 1))
                ed_dmma<M, D, GREC>(dv, in, out, e, vrec, frec, s_orient, opbuf_base, gv0, gv1, fp0, fp1, first);
            ed_stream<D>(dv, in, out, e, vrec, frec, s_orient, opbuf_base, s_bars, ed_streamed && !(dbg_skip & 1), hs && !(dbg_skip & 2), split_copies);
            if (hs) hgf_done = j_done = true;
            dbg_skip |= 1;
        }
    }
    if constexpr (ED && GREC && M > 1 && D == 3 && (NT == 256 || NT == 512)) {
        if (ed_streamed && !(dbg_skip & 1)) {  // wide system, pe = 64: one streamed sweep per component pair, then the face blocks
            const bool want_hgf = hgf_streamed && ed_dmma_on == 2 && !(dbg_skip & 2);
            if (want_hgf && NT == 256 && pf == 16 && qf <= 32) {
                // J outside the per-face diagonal blocks is zero (the face stages write the blocks themselves)
                for (int t = tid; t < nfl * nfl; t += nt) {
                    const int c = t / nfl, r = t - c * nfl;
                    if (c / mpf != r / mpf) out.J[static_cast<size_t>(e) * nfl * nfl + t] = 0.0;
                }
            }
            if (ed_stream_wide<M, D, NT / 32>(dv, in, out, e, vrec, frec, s_orient, opbuf_base, s_bars, want_hgf)) hgf_done = j_done = true;
            dbg_skip |= 1;
        }
    }
    if (ED && ed_dmma_on && !(dbg_skip & 1)) {
        // operand chunks live behind the point records (16-byte aligned)
        double* opbuf = opbuf_base;
        ed_dmma<M, D, GREC>(dv, in, out, e, vrec, frec, s_orient, opbuf, gv0, gv1, fp0, fp1, first);
    } else if (!(dbg_skip & 1)) {
        constexpr int TI = (M == 1) ? 2 : 1, TJ = (M == 1) ? 4 : 1;
        constexpr int Q = M * (1 + D);  // per row component m: E then D_0..D_{D-1}
        const int nti = (pe + TI - 1) / TI, ntj = (pe + TJ - 1) / TJ;
        for (int t = tid; t < nti * ntj; t += nt) {
            const int bj = t / nti, bi = t - bj * nti;
            for (int mp = 0; mp < M; ++mp) {
                double acc[TI][TJ][Q];
#pragma unroll
                for (int a = 0; a < TI; ++a)
#pragma unroll
                    for (int b = 0; b < TJ; ++b)
#pragma unroll
                        for (int q = 0; q < Q; ++q) acc[a][b][q] = 0.0;
                for (int g = gv0; g < gv1; ++g) {
                    const VR& r = vrec[g - gv0];
                    double val[TI][Q];
#pragma unroll
                    for (int a = 0; a < TI; ++a) {
                        const int i = min(bi * TI + a, pe - 1);
                        const double phi_i = dv.phi[i + pe * g];
                        double dp_[D];
#pragma unroll
                        for (int k = 0; k < D; ++k) dp_[k] = dv.dphi[k][i + pe * g];
#pragma unroll
                        for (int m = 0; m < M; ++m) {
                            const int mm = m * M + mp;
                            double fe = 0.0;
#pragma unroll
                            for (int k = 0; k < D; ++k) fe += r.cE[mm * D + k] * dp_[k];
                            double eij = -fe - r.dSu[mm] * phi_i;
                            if (transient && m == mp) eij += in.dt_inv * phi_i;
                            val[a][m] = eij;
#pragma unroll
                            for (int dp = 0; dp < D; ++dp) {
                                double fd = 0.0;
#pragma unroll
                                for (int k = 0; k < D; ++k) fd += r.cD[(dp * M * M + mm) * D + k] * dp_[k];
                                val[a][M * (1 + dp) + m] = -fd - r.dSq[mm * D + dp] * phi_i;
                            }
                        }
                    }
#pragma unroll
                    for (int b = 0; b < TJ; ++b) {
                        const int j = min(bj * TJ + b, pe - 1);
                        const double pj = r.w * dv.phi[j + pe * g];
#pragma unroll
                        for (int a = 0; a < TI; ++a)
#pragma unroll
                            for (int q = 0; q < Q; ++q) acc[a][b][q] = fma(pj, val[a][q], acc[a][b][q]);
                    }
                }
                for (int p = fp0; p < fp1; ++p) {
                    const int lf = p / qf, gc = p - lf * qf;
                    const FR& r = frec[p - fp0];
                    const double* phis = dv.tphi + ((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe;
                    double val[TI][Q];
#pragma unroll
                    for (int a = 0; a < TI; ++a) {
                        const double ph = phis[min(bi * TI + a, pe - 1)];
#pragma unroll
                        for (int m = 0; m < M; ++m) {
                            val[a][m] = (m == mp) ? r.tau * ph : 0.0;
#pragma unroll
                            for (int dp = 0; dp < D; ++dp) val[a][M * (1 + dp) + m] = r.dfh_q[(m * M + mp) * D + dp] * ph;
                        }
                    }
#pragma unroll
                    for (int b = 0; b < TJ; ++b) {
                        const double pj = r.w * phis[min(bj * TJ + b, pe - 1)];
#pragma unroll
                        for (int a = 0; a < TI; ++a)
#pragma unroll
                            for (int q = 0; q < Q; ++q) acc[a][b][q] = fma(pj, val[a][q], acc[a][b][q]);
                    }
                }
#pragma unroll
                for (int a = 0; a < TI; ++a)
#pragma unroll
                    for (int b = 0; b < TJ; ++b) {
                        const int i = bi * TI + a, j = bj * TJ + b;
                        if (i >= pe || j >= pe) continue;
                        for (int m = 0; m < M; ++m) {
                            const size_t o = static_cast<size_t>(e) * npe * npe + static_cast<size_t>(mp * pe + j) * npe + (m * pe + i);
                            if (first) {
                                out.E[o] = acc[a][b][m];
                                for (int dp = 0; dp < D; ++dp) out.Dm[dp][o] = acc[a][b][M * (1 + dp) + m];
                            } else {
                                out.E[o] += acc[a][b][m];
                                for (int dp = 0; dp < D; ++dp) out.Dm[dp][o] += acc[a][b][M * (1 + dp) + m];
                            }
                        }
                    }
            }
        }
    }
    if constexpr (ED) {
        if (hgf_done) {
        } else if (ed_dmma_on == 2 && (dbg_skip & 2)) hgf_done = true;
        else if (ed_dmma_on == 2) {  // all face points in this launch, every output entry written exactly once
            double* opbuf = opbuf_base;
            hgf_dmma<M, D, GREC>(dv, out, e, frec, s_orient, opbuf);
            hgf_done = true;
        }
    }
    // ---- H and G_d: rows (lf, m, b), columns (mp, j) ----
    for (int t = tid; t < (hgf_done ? 0 : n_lfe * pf * pe); t += nt) {
        const int j = t / (n_lfe * pf);
        const int lb = t - j * (n_lfe * pf);
        const int lf = lb / pf, b = lb - lf * pf;
        double aH[M * M], aG[D * M * M];
        for (int k = 0; k < M * M; ++k) aH[k] = 0.0;
        for (int k = 0; k < D * M * M; ++k) aG[k] = 0.0;
        const int g0 = max(0, fp0 - lf * qf), g1 = min(qf, fp1 - lf * qf);
        if (!first && g0 >= g1) continue;
        for (int gc = g0; gc < g1; ++gc) {
            const FR& r = frec[lf * qf + gc - fp0];
            const double pj = r.w * dv.tphi[((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe + j];
            const double ps = dv.psi[b + pf * gc];
            for (int k = 0; k < M * M; ++k) {
                aH[k] += pj * r.dv_u[k] * ps;
                for (int dp = 0; dp < D; ++dp) aG[dp * M * M + k] += pj * r.dv_q[k * D + dp] * ps;
            }
        }
        for (int m = 0; m < M; ++m)
            for (int mp = 0; mp < M; ++mp) {
                const size_t o = static_cast<size_t>(e) * nfl * npe + static_cast<size_t>(mp * pe + j) * nfl + (lf * mpf + m * pf + b);
                if (first) {
                    out.H[o] = aH[m * M + mp];
                    for (int dp = 0; dp < D; ++dp) out.G[dp][o] = aG[dp * M * M + m * M + mp];
                } else {
                    out.H[o] += aH[m * M + mp];
                    for (int dp = 0; dp < D; ++dp) out.G[dp][o] += aG[dp * M * M + m * M + mp];
                }
            }
    }
    // ---- F: rows (m, i), columns (lf, mp, bp) ----
    for (int t = tid; t < (hgf_done ? 0 : pe * n_lfe * pf); t += nt) {
        const int lb = t / pe, i = t - lb * pe;
        const int lf = lb / pf, bp = lb - lf * pf;
        double aF[M * M];
        for (int k = 0; k < M * M; ++k) aF[k] = 0.0;
        const int g0 = max(0, fp0 - lf * qf), g1 = min(qf, fp1 - lf * qf);
        if (!first && g0 >= g1) continue;
        for (int gc = g0; gc < g1; ++gc) {
            const FR& r = frec[lf * qf + gc - fp0];
            const double pj = r.w * dv.psi[bp + pf * gc];
            const double ph = dv.tphi[((static_cast<size_t>(lf) * dv.n_orient + s_orient[lf]) * qf + gc) * pe + i];
            for (int k = 0; k < M * M; ++k) aF[k] += pj * r.dfh_uh[k] * ph;
        }
        for (int m = 0; m < M; ++m)
            for (int mp = 0; mp < M; ++mp) {
                double* o = out.F + static_cast<size_t>(e) * npe * nfl + static_cast<size_t>(lf * mpf + mp * pf + bp) * npe + (m * pe + i);
                *o = first ? aF[m * M + mp] : *o + aF[m * M + mp];
            }
    }
    // ---- J: block diagonal over local faces; rows (lf, m, b), columns (lf, mp, bp); the other
    // entries of the nfl x nfl block are zero ----
    if (j_done) return;
    if (first)
        for (int t = tid; t < nfl * nfl; t += nt) out.J[static_cast<size_t>(e) * nfl * nfl + t] = 0.0;
    __syncthreads();
    for (int t = tid; t < n_lfe * pf * pf; t += nt) {
        const int lf = t / (pf * pf);
        const int r2 = t - lf * pf * pf;
        const int bp = r2 / pf, b = r2 - bp * pf;
        double aJ[M * M];
        for (int k = 0; k < M * M; ++k) aJ[k] = 0.0;
        const int g0 = max(0, fp0 - lf * qf), g1 = min(qf, fp1 - lf * qf);
        if (!first && g0 >= g1) continue;
        for (int gc = g0; gc < g1; ++gc) {
            const FR& r = frec[lf * qf + gc - fp0];
            const double pj = r.w * dv.psi[bp + pf * gc];
            const double ps = dv.psi[b + pf * gc];
            for (int k = 0; k < M * M; ++k) aJ[k] += pj * r.dv_uh[k] * ps;
        }
        for (int m = 0; m < M; ++m)
            for (int mp = 0; mp < M; ++mp) {
                double* o = out.J + static_cast<size_t>(e) * nfl * nfl + static_cast<size_t>(lf * mpf + mp * pf + bp) * nfl + (lf * mpf + m * pf + b);
                *o = first ? aJ[m * M + mp] : *o + aJ[m * M + mp];
            }
    }
}

template <class Model>
void launch_assemble_t(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in,
                       const LocalOut& out, bool want_jac) {
    constexpr int M = Model::M, D = Model::D;
    const int npe = M * dv.pe, nfl = dv.n_lfe * M * dv.pf;
    const int nfp = dv.n_lfe * dv.qf;
    const size_t fixed = (static_cast<size_t>(npe) * (2 + D + kResParts) + nfl) * sizeof(double);
    const size_t cap = 216 * 1024;
    const size_t budget = std::min<size_t>(cap, static_cast<size_t>(tuning().assemble_budget_kb) * 1024);
    const size_t svr = sizeof(VolRec<M, D>), sfr = sizeof(FaceRec<M, D>);
    if (fixed + std::max(svr, sfr) > budget)
        throw Failure(HDGB_ERR_UNSUPPORTED, "local assembly: element state exceeds shared memory");
    auto kern = local_assemble_kernel<Model, 256, false, false>;
    auto kern_r = local_assemble_kernel<Model, 256, false, false, true>;  // residual only
    constexpr int NTD = 256;  // tensor-core mode: 8 warps, two CTAs per SM for scalar systems (their phases overlap)
    auto kern_d = local_assemble_kernel<Model, NTD, true, false>;
    ensure_dynamic_smem(kern, cap);
    ensure_dynamic_smem(kern_r, cap);
    ensure_dynamic_smem(kern_d, cap);
    const size_t all = fixed + dv.qe * svr + nfp * sfr;
    if (all <= budget) {
        // E / D_d on the tensor-core path when the operand chunks fit next to the point records
        size_t ed_bytes = 2 * ed_plan(dv.pe, M, D, NTD / 32).doubles(D) * sizeof(double) + 16;
        ed_bytes = std::max(ed_bytes, hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M) * sizeof(double) + 16);
        const bool ed = want_jac && tuning().use_dmma && ed_dmma_ok(dv.pe, M, D) && hgf_dmma_ok(dv.pf, dv.qf) && all + ed_bytes <= cap;
        // 16-warp variant (one CTA per SM): all 1 + D matrices of a scalar system in ONE point sweep
        if constexpr (M == 1 && D == 3) {  // (instantiated for the 3D models only: build time)
            if (ed && tuning().local_nt == 512) {
                const EdPlan p16 = ed_plan(dv.pe, M, D, 16);
                const size_t eb = std::max(2 * p16.doubles(D), hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M)) * sizeof(double) + 16;
                if (p16.wsub <= 4 && all + eb <= cap) {
                    auto kern_w = local_assemble_kernel<Model, 512, true, false>;
                    ensure_dynamic_smem(kern_w, cap);
                    kern_w<<<dv.ne, 512, all + eb, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 2 | (tuning().local_debug_skip << 4), nullptr, 0);
                    HDGB_LAUNCH_CHECK(ctx);
                    return;
                }
            }
        }
        if (ed && ed_stream_ok(dv, M)) {
            const size_t es_bytes = std::max(ed_stream_doubles(D), hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M)) * sizeof(double) + 16;
            if (all + es_bytes <= cap) {
                kern_d<<<dv.ne, NTD, all + es_bytes, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 2 | ((tuning().local_ed_stream & 1) ? 8 : 0) | ((tuning().local_ed_stream & 2) ? 128 : 0) | ((tuning().local_ed_stream & 4) ? 256 : 0) | ((tuning().local_debug_skip & 7) << 4), nullptr, 0);
                HDGB_LAUNCH_CHECK(ctx);
                return;
            }
        }
        if (ed) kern_d<<<dv.ne, NTD, all + ed_bytes, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 2 | (tuning().local_debug_skip << 4), nullptr, 0);
        else if (!want_jac) kern_r<<<dv.ne, 256, all, ctx->stream>>>(dv, mv, in, out, 0, 0, dv.qe, 0, nfp, 1, 0, nullptr, 0);
        else kern<<<dv.ne, 256, all, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 0, nullptr, 0);
        HDGB_LAUNCH_CHECK(ctx);
        return;
    }
    // wide systems with the Jacobian on the tensor-core path: records in a global (L2) scratch, one launch
    if constexpr (M > 1) {
        if (want_jac && tuning().use_dmma && tuning().local_global_records && ed_dmma_ok(dv.pe, M, D) && hgf_dmma_ok(dv.pf, dv.qf)) {
            const size_t rec_stride = (dv.qe * svr + nfp * sfr + 15) & ~static_cast<size_t>(15);
            // 16 warps: two component pairs share one point sweep (and one weighted-basis operand)
            const EdPlan p16 = ed_plan(dv.pe, M, D, 16);
            const size_t edb16 = std::max(2 * p16.doubles(D), hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M)) * sizeof(double) + 32;
            if constexpr (D == 3) {
                const bool wide_stream = dv.pe == kEsPe && dv.es_vol && (tuning().local_ed_stream & 1);
                const size_t edw16 = std::max(ed_wide_doubles(D, dv.qe, nfp), hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M)) * sizeof(double) + 32;
                // streamed sweep with 16 warps (each warp half the columns): measured slower than 8 warps (config 5 at 12^3: 32.8 vs 31.4 ms -- the
                // left fragments are formed twice), kept behind local_nt_wide = 512
                if (wide_stream && tuning().local_nt_wide == 512 && fixed + edw16 <= cap) {
                    auto kern_gw = local_assemble_kernel<Model, 512, true, true>;
                    ensure_dynamic_smem(kern_gw, cap);
                    DevBuf<char> scratch(rec_stride * static_cast<size_t>(dv.ne));
                    kern_gw<<<dv.ne, 512, fixed + edw16, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 2 | 8 | ((tuning().local_debug_skip & 7) << 4), scratch.p, rec_stride);
                    HDGB_LAUNCH_CHECK(ctx);
                    return;
                }
                if (tuning().local_nt == 512 && p16.wsub <= 8 && fixed + edb16 <= cap) {
                    auto kern_gw = local_assemble_kernel<Model, 512, true, true>;
                    ensure_dynamic_smem(kern_gw, cap);
                    DevBuf<char> scratch(rec_stride * static_cast<size_t>(dv.ne));
                    kern_gw<<<dv.ne, 512, fixed + edb16, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 2 | (tuning().local_debug_skip << 4), scratch.p, rec_stride);
                    HDGB_LAUNCH_CHECK(ctx);
                    return;
                }
            }
            size_t edb = std::max(2 * ed_plan(dv.pe, M, D, 8).doubles(D), hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M)) * sizeof(double) + 32;
            int stream_flag = 0;
            if (D == 3 && dv.pe == kEsPe && dv.es_vol && (tuning().local_ed_stream & 1)) {
                const size_t edw = std::max(ed_wide_doubles(D, dv.qe, nfp), hgf_plan(dv.pe, dv.pf, dv.qf).doubles(D, M)) * sizeof(double) + 32;
                if (fixed + edw <= cap) { edb = edw; stream_flag = 8; }
            }
            if (fixed + edb <= cap) {
                auto kern_g = local_assemble_kernel<Model, 256, true, true>;
                ensure_dynamic_smem(kern_g, cap);
                DevBuf<char> scratch(rec_stride * static_cast<size_t>(dv.ne));
                kern_g<<<dv.ne, 256, fixed + edb, ctx->stream>>>(dv, mv, in, out, 1, 0, dv.qe, 0, nfp, 1, 2 | stream_flag | ((stream_flag && (tuning().local_ed_stream & 2)) ? 128 : 0) | ((tuning().local_debug_skip & 7) << 4), scratch.p, rec_stride);
                HDGB_LAUNCH_CHECK(ctx);
                return;
            }
        }
    }
    // point-chunked sweep: volume chunks first, then face chunks (the reference's accumulation order).  With
    // the Jacobian on the tensor-core path the operand tiles share the budget with the point records.
    size_t ed_bytes = 0;
    // (measured on config 5: the 50 operand passes per launch cost more than the scalar sweep saves -- off by default)
    if (want_jac && tuning().use_dmma && tuning().local_dmma_chunked && ed_dmma_ok(dv.pe, M, D)) {
        ed_bytes = 2 * ed_plan(dv.pe, M, D, NTD / 32).doubles(D) * sizeof(double) + 16;
        if (fixed + ed_bytes + 8 * std::max(svr, sfr) > budget) ed_bytes = 0;
    }
    const int edf = ed_bytes ? 1 : 0;
    const int vc = static_cast<int>((budget - fixed - ed_bytes) / svr), fc = static_cast<int>((budget - fixed - ed_bytes) / sfr);
    int first = 1;
    for (int g0 = 0; g0 < dv.qe; g0 += vc) {
        const int g1 = std::min(dv.qe, g0 + vc);
        const size_t sm_b = fixed + (g1 - g0) * svr + ed_bytes;
        if (edf) kern_d<<<dv.ne, NTD, sm_b, ctx->stream>>>(dv, mv, in, out, 1, g0, g1, 0, 0, first, 1, nullptr, 0);
        else if (!want_jac) kern_r<<<dv.ne, 256, sm_b, ctx->stream>>>(dv, mv, in, out, 0, g0, g1, 0, 0, first, 0, nullptr, 0);
        else kern<<<dv.ne, 256, sm_b, ctx->stream>>>(dv, mv, in, out, 1, g0, g1, 0, 0, first, 0, nullptr, 0);
        HDGB_LAUNCH_CHECK(ctx);
        first = 0;
    }
    for (int p0 = 0; p0 < nfp; p0 += fc) {
        const int p1 = std::min(nfp, p0 + fc);
        const size_t sm_b = fixed + (p1 - p0) * sfr + ed_bytes;
        if (edf) kern_d<<<dv.ne, NTD, sm_b, ctx->stream>>>(dv, mv, in, out, 1, 0, 0, p0, p1, first, 1, nullptr, 0);
        else if (!want_jac) kern_r<<<dv.ne, 256, sm_b, ctx->stream>>>(dv, mv, in, out, 0, 0, 0, p0, p1, first, 0, nullptr, 0);
        else kern<<<dv.ne, 256, sm_b, ctx->stream>>>(dv, mv, in, out, 1, 0, 0, p0, p1, first, 0, nullptr, 0);
        HDGB_LAUNCH_CHECK(ctx);
        first = 0;
    }
}

}  // namespace

// The model instantiations are split over three translation units (this file compiled with
// -DHDGB_LOCAL_PART=0|1|2, see the Makefile) so that they build in parallel.
#ifndef HDGB_LOCAL_PART
#define HDGB_LOCAL_PART 0
#endif
void launch_local_assemble_part1(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in, const LocalOut& out, bool want_jac);
void launch_local_assemble_part2(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in, const LocalOut& out, bool want_jac);

#if HDGB_LOCAL_PART == 0
void launch_local_factors(hdgb_ctx* ctx, const DiscView& dv, double* mass, double* const bmat[3], double* const cmat[3]) {
    const size_t sm_m = static_cast<size_t>(dv.qe) * (1 + dv.D * dv.D) * sizeof(double);
    const size_t sm_c = static_cast<size_t>(dv.n_lfe) * dv.qf * (1 + dv.D) * sizeof(double);
    if (dv.D == 2) {
        ensure_dynamic_smem(mass_bmat_kernel<2>, sm_m);
        mass_bmat_kernel<2><<<dv.ne, 256, sm_m, ctx->stream>>>(dv, mass, bmat[0], bmat[1], bmat[2]);
        HDGB_LAUNCH_CHECK(ctx);
        cmat_kernel<2><<<dv.ne, 256, sm_c, ctx->stream>>>(dv, cmat[0], cmat[1], cmat[2]);
    } else {
        ensure_dynamic_smem(mass_bmat_kernel<3>, sm_m);
        mass_bmat_kernel<3><<<dv.ne, 256, sm_m, ctx->stream>>>(dv, mass, bmat[0], bmat[1], bmat[2]);
        HDGB_LAUNCH_CHECK(ctx);
        cmat_kernel<3><<<dv.ne, 256, sm_c, ctx->stream>>>(dv, cmat[0], cmat[1], cmat[2]);
    }
    HDGB_LAUNCH_CHECK(ctx);
}

void launch_local_assemble(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in,
                           const LocalOut& out, bool want_jac) {
    if (dv.n_lfe > 8) throw Failure(HDGB_ERR_UNSUPPORTED, "local assembly: more than 8 local faces");
    const int D = dv.D;
    switch (mv.kind) {
        case HDGB_MODEL_POISSON:
            if (D == 2) launch_assemble_t<PoissonModel<2>>(ctx, dv, mv, in, out, want_jac);
            else launch_assemble_t<PoissonModel<3>>(ctx, dv, mv, in, out, want_jac);
            break;
        case HDGB_MODEL_REACTION:
            if (D == 2) launch_assemble_t<ReactionModel<2>>(ctx, dv, mv, in, out, want_jac);
            else launch_assemble_t<ReactionModel<3>>(ctx, dv, mv, in, out, want_jac);
            break;
        case HDGB_MODEL_BURGERS:
        case HDGB_MODEL_CONVDIFF:
            launch_local_assemble_part1(ctx, dv, mv, in, out, want_jac);
            break;
        case HDGB_MODEL_ELASTICITY:
        case HDGB_MODEL_NAVIER_STOKES:
            launch_local_assemble_part2(ctx, dv, mv, in, out, want_jac);
            break;
        default:
            throw Failure(HDGB_ERR_UNSUPPORTED, "unknown model kind " + std::to_string(mv.kind));
    }
}
#elif HDGB_LOCAL_PART == 1
void launch_local_assemble_part1(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in,
                                 const LocalOut& out, bool want_jac) {
    const int D = dv.D;
    if (mv.kind == HDGB_MODEL_BURGERS) {
        if (D == 2) launch_assemble_t<BurgersModel<2>>(ctx, dv, mv, in, out, want_jac);
        else launch_assemble_t<BurgersModel<3>>(ctx, dv, mv, in, out, want_jac);
    } else {
        if (D == 2) launch_assemble_t<ConvDiffModel<2>>(ctx, dv, mv, in, out, want_jac);
        else launch_assemble_t<ConvDiffModel<3>>(ctx, dv, mv, in, out, want_jac);
    }
}
#else
void launch_local_assemble_part2(hdgb_ctx* ctx, const DiscView& dv, const ModelView& mv, const LocalIn& in,
                                 const LocalOut& out, bool want_jac) {
    const int D = dv.D;
    if (mv.kind == HDGB_MODEL_ELASTICITY) {
        if (D == 2) launch_assemble_t<ElasticityModel<2>>(ctx, dv, mv, in, out, want_jac);
        else launch_assemble_t<ElasticityModel<3>>(ctx, dv, mv, in, out, want_jac);
    } else {
        if (D == 2) launch_assemble_t<NavierStokesModel<2>>(ctx, dv, mv, in, out, want_jac);
        else launch_assemble_t<NavierStokesModel<3>>(ctx, dv, mv, in, out, want_jac);
    }
}
#endif

}  // namespace hdgb
