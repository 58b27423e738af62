// hw_acoustic.cu — acoustic p-v leapfrog phase kernels (sm_100a), any lanes, 2D/3D.
//
// Per step n (AcousticSolver._step_work, acoustic.py:162-181):
//   velocity phase  vx, v_slow(, v_mid) from p^n    -> k_ac_vel
//   pressure phase  p from div v^{n+1/2} + source    -> k_ac_pres (+ fused fp64 energy
//                   partials on sample steps, diagnostics.py:76-87)
// One thread owns W consecutive x cells of one (slow, mid) row; every tap address
// is the thread's precomputed cell offset plus a constant (Cell, hw_common.cuh).
// (The binary16 2D case runs in the fused single-pass kernel, hw_fused2d.cu.)
#include "hw_params.h"

namespace hw {

template <int LU, int W>
__device__ __forceinline__ void upd_store(const FieldView& f, const FieldView& rf, const Cell& c, int64_t s,
                                          vec<LU, W> u, vec<LU, W> rr, bool comp, unsigned int& mask) {
    store_c<LU, W>(f, c, s, u);
    if (!vfinite<LU, W>(u)) mask |= 1u << f.bit;
    if (comp) {
        store_c<LU, W>(rf, c, s, rr);
        if (!vfinite<LU, W>(rr)) mask |= 1u << rf.bit;
    }
}

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK, 8) k_ac_vel(AcParams P, int64_t n) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    const Geom& g = P.g;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    unsigned int mask = 0;
    if (xv * W < g.nx && s < P.p.rows) {
        const Cell c = make_cell(g, s, m, xv * W);
        TS k[4];
#pragma unroll
        for (int j = 0; j < 4; j++) k[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        const TU* pp = fptr<TU>(P.p, c);
        vec<LU, W> t[4];
        // vx = fl(fl(ddx p / rho_x) * dt), advance (acoustic.py:167-168)
        xtaps_c<LU, W>(pp, c, false, t);
        {
            vec<LU, W> u = vload<LU, W>(fptr<TU>(P.vx, c));
            vec<LU, W> rr = comp ? vload<LU, W>(fptr<TU>(P.rvx, c)) : vec<LU, W>{};
            finish<LS, LU, W>(fold<LS, LU, W>(k, t, P.order), &P.rho_x, s, m, xv * W, dt, P.variant, -1, 0.0, u, rr);
            upd_store<LU, W>(P.vx, P.rvx, c, s, u, rr, comp, mask);
        }
        // v_slow from dds p (acoustic.py:169-170)
        staps_c<LU, W>(pp, c, false, P.order, t);
        {
            vec<LU, W> u = vload<LU, W>(fptr<TU>(P.vs, c));
            vec<LU, W> rr = comp ? vload<LU, W>(fptr<TU>(P.rvs, c)) : vec<LU, W>{};
            finish<LS, LU, W>(fold<LS, LU, W>(k, t, P.order), &P.rho_s, s, m, xv * W, dt, P.variant, -1, 0.0, u, rr);
            upd_store<LU, W>(P.vs, P.rvs, c, s, u, rr, comp, mask);
        }
        if (P.d3) {  // v_mid from ddm p (3D extension)
            mtaps_c<LU, W>(pp, c, false, P.order, t);
            vec<LU, W> u = vload<LU, W>(fptr<TU>(P.vm, c));
            vec<LU, W> rr = comp ? vload<LU, W>(fptr<TU>(P.rvm, c)) : vec<LU, W>{};
            finish<LS, LU, W>(fold<LS, LU, W>(k, t, P.order), &P.rho_m, s, m, xv * W, dt, P.variant, -1, 0.0, u, rr);
            upd_store<LU, W>(P.vm, P.rvm, c, s, u, rr, comp, mask);
        }
    }
    record_failure(P.ctrl, n, mask);
}

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK, 8) k_ac_pres(AcParams P, int64_t n, double src, int sample) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    const Geom& g = P.g;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    unsigned int mask = 0;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (xv * W < g.nx && s < P.p.rows) {
        const int64_t x = xv * W;
        const Cell c = make_cell(g, s, m, x);
        TS k[4];
#pragma unroll
        for (int j = 0; j < 4; j++) k[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        using OS = vops<LS, W>;
        vec<LU, W> tx[4], ts[4], tm[4];
        // divergence fl(fl(ddx vx + dds vs) + ddm vm) (acoustic.py:172-175)
        xtaps_c<LU, W>(fptr<TU>(P.vx, c), c, true, tx);
        staps_c<LU, W>(fptr<TU>(P.vs, c), c, true, P.order, ts);
        vec<LS, W> div = OS::add(fold<LS, LU, W>(k, tx, P.order), fold<LS, LU, W>(k, ts, P.order));
        if (P.d3) {
            mtaps_c<LU, W>(fptr<TU>(P.vm, c), c, true, P.order, tm);
            div = OS::add(div, fold<LS, LU, W>(k, tm, P.order));
        }
        int src_lane = -1;
        if (P.has_src && s == P.src_s && m == P.src_m && P.src_x >= x && P.src_x < x + W)
            src_lane = (int)(P.src_x - x);
        const vec<LU, W> p_old = vload<LU, W>(fptr<TU>(P.p, c));
        vec<LU, W> u = p_old;
        vec<LU, W> rr = comp ? vload<LU, W>(fptr<TU>(P.rp, c)) : vec<LU, W>{};
        finish<LS, LU, W>(div, &P.beta, s, m, x, dt, P.variant, src_lane, src, u, rr);
        upd_store<LU, W>(P.p, P.rp, c, s, u, rr, comp, mask);
        if (sample) {  // E = dx^2/2 [sum beta p^n p^{n+1} + sum rho v^2] (diagnostics.py:76-87)
#pragma unroll
            for (int i = 0; i < W; i++) {
                const int64_t xi = x + i;
                double po = lane<LU>::to_f64(p_old.e[i]), pn = lane<LU>::to_f64(u.e[i]);
                double vxv = lane<LU>::to_f64(tx[2].e[i]), vsv = lane<LU>::to_f64(ts[2].e[i]);
                e[0] += p64(P.e_beta, s, m, xi) * (po * pn);
                e[1] += p64(P.e_rho_x, s, m, xi) * (vxv * vxv);
                e[2] += p64(P.e_rho_s, s, m, xi) * (vsv * vsv);
                if (P.d3) {
                    double vmv = lane<LU>::to_f64(tm[2].e[i]);
                    e[3] += p64(P.e_rho_m, s, m, xi) * (vmv * vmv);
                }
            }
        }
    }
    record_failure(P.ctrl, n, mask);
    if (sample) block_partials(e, P.partials);
}

// E(t=0): the state paired with itself (acoustic.py:205-208).
template <int LU, int W>
__global__ void __launch_bounds__(BLOCK, 8) k_ac_energy(AcParams P) {
    using TU = typename lane<LU>::T;
    const Geom& g = P.g;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (xv * W < g.nx && s < P.p.rows) {
        const int64_t x = xv * W;
        const Cell c = make_cell(g, s, m, x);
        vec<LU, W> p = vload<LU, W>(fptr<TU>(P.p, c));
        vec<LU, W> vx = vload<LU, W>(fptr<TU>(P.vx, c));
        vec<LU, W> vs = vload<LU, W>(fptr<TU>(P.vs, c));
#pragma unroll
        for (int i = 0; i < W; i++) {
            const int64_t xi = x + i;
            double pv = lane<LU>::to_f64(p.e[i]);
            double a = lane<LU>::to_f64(vx.e[i]), b = lane<LU>::to_f64(vs.e[i]);
            e[0] += p64(P.e_beta, s, m, xi) * (pv * pv);
            e[1] += p64(P.e_rho_x, s, m, xi) * (a * a);
            e[2] += p64(P.e_rho_s, s, m, xi) * (b * b);
        }
        if (P.d3) {
            vec<LU, W> vm = vload<LU, W>(fptr<TU>(P.vm, c));
#pragma unroll
            for (int i = 0; i < W; i++) {
                double a = lane<LU>::to_f64(vm.e[i]);
                e[3] += p64(P.e_rho_m, s, m, x + i) * (a * a);
            }
        }
    }
    block_partials(e, P.partials);
}

// ------------------------------------------------------------------ launchers

void launch_ac_vel(int LS, int LU, int W, const AcParams& P, int64_t n, int64_t nblocks, cudaStream_t st) {
    HW_DISPATCH_LS(LS, HW_DISPATCH_LU(LU, HW_DISPATCH_W(W, k_ac_vel<LS_, LU_, W_><<<grid3(P.g, W, nblocks), block3(P.g, W), 0, st>>>(P, n))))
}
void launch_ac_pres(int LS, int LU, int W, const AcParams& P, int64_t n, double src, int sample, int64_t nblocks,
                    cudaStream_t st) {
    HW_DISPATCH_LS(LS, HW_DISPATCH_LU(LU, HW_DISPATCH_W(W, k_ac_pres<LS_, LU_, W_><<<grid3(P.g, W, nblocks), block3(P.g, W), 0, st>>>(P, n, src, sample))))
}
void launch_ac_energy(int LU, int W, const AcParams& P, int64_t nblocks, cudaStream_t st) {
    HW_DISPATCH_LU(LU, HW_DISPATCH_W(W, k_ac_energy<LU_, W_><<<grid3(P.g, W, nblocks), block3(P.g, W), 0, st>>>(P)))
}

}  // namespace hw
