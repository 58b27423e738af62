// hw_acoustic.cu — acoustic p-v leapfrog phase kernels (sm_100a).
//
// Per step n (AcousticSolver._step_work, acoustic.py:162-181):
//   velocity phase  vx, vy(, vz) from p^n         -> k_ac_vel
//   pressure phase  p from div v^{n+1/2} + source -> k_ac_pres (+ fused fp64 energy
//                   partials on sample steps, diagnostics.py:76-87)
// One thread owns W consecutive x cells of one (slow, mid) row; all loads and
// stores are W-wide and coalesced along x.
#include "hw_params.h"

namespace hw {

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK) k_ac_vel(AcParams P, int64_t n) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    const Geom& g = P.g;
    const int64_t nxv = g.nx / W;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    unsigned int mask = 0;
    if (xv < nxv && s < P.p.rows) {
        const int64_t x = xv * W;
        TS c[4];
#pragma unroll
        for (int j = 0; j < 4; j++) c[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        vec<LU, W> t[4];
        // vx = fl(fl(ddx p / rho_x) * dt), advance (acoustic.py:167-168)
        xtaps<LU, W>(frow<TU>(P.p, g, s, m), x, g.nx, false, t);
        {
            vec<LS, W> d = fold<LS, LU, W>(c, t, P.order);
            vec<LU, W> u = vload<LU, W>(frow<TU>(P.vx, g, s, m) + x);
            vec<LU, W> rr = comp ? vload<LU, W>(frow<TU>(P.rvx, g, s, m) + x) : vec<LU, W>{};
            finish<LS, LU, W>(d, &P.rho_x, s, m, x, dt, P.variant, -1, 0.0, u, rr);
            store_field<LU, W>(P.vx, g, s, m, x, u);
            if (!vfinite<LU, W>(u)) mask |= 1u << P.vx.bit;
            if (comp) {
                store_field<LU, W>(P.rvx, g, s, m, x, rr);
                if (!vfinite<LU, W>(rr)) mask |= 1u << P.rvx.bit;
            }
        }
        // v_slow from dds p (acoustic.py:169-170)
        staps<LU, W>(P.p, g, s, m, x, false, P.order, t);
        {
            vec<LS, W> d = fold<LS, LU, W>(c, t, P.order);
            vec<LU, W> u = vload<LU, W>(frow<TU>(P.vs, g, s, m) + x);
            vec<LU, W> rr = comp ? vload<LU, W>(frow<TU>(P.rvs, g, s, m) + x) : vec<LU, W>{};
            finish<LS, LU, W>(d, &P.rho_s, s, m, x, dt, P.variant, -1, 0.0, u, rr);
            store_field<LU, W>(P.vs, g, s, m, x, u);
            if (!vfinite<LU, W>(u)) mask |= 1u << P.vs.bit;
            if (comp) {
                store_field<LU, W>(P.rvs, g, s, m, x, rr);
                if (!vfinite<LU, W>(rr)) mask |= 1u << P.rvs.bit;
            }
        }
        if (P.d3) {  // v_mid from ddm p (3D extension)
            mtaps<LU, W>(P.p, g, s, m, x, false, P.order, t);
            vec<LS, W> d = fold<LS, LU, W>(c, t, P.order);
            vec<LU, W> u = vload<LU, W>(frow<TU>(P.vm, g, s, m) + x);
            vec<LU, W> rr = comp ? vload<LU, W>(frow<TU>(P.rvm, g, s, m) + x) : vec<LU, W>{};
            finish<LS, LU, W>(d, &P.rho_m, s, m, x, dt, P.variant, -1, 0.0, u, rr);
            store_field<LU, W>(P.vm, g, s, m, x, u);
            if (!vfinite<LU, W>(u)) mask |= 1u << P.vm.bit;
            if (comp) {
                store_field<LU, W>(P.rvm, g, s, m, x, rr);
                if (!vfinite<LU, W>(rr)) mask |= 1u << P.rvm.bit;
            }
        }
    }
    record_failure(P.ctrl, n, mask);
}

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK) k_ac_pres(AcParams P, int64_t n, double src, int sample) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    const Geom& g = P.g;
    const int64_t nxv = g.nx / W;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    unsigned int mask = 0;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (xv < nxv && s < P.p.rows) {
        const int64_t x = xv * W;
        TS c[4];
#pragma unroll
        for (int j = 0; j < 4; j++) c[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        using OS = vops<LS, W>;
        vec<LU, W> tx[4], ts[4], tm[4];
        // divergence fl(fl(ddx vx + dds vs) + ddm vm) (acoustic.py:172-175)
        xtaps<LU, W>(frow<TU>(P.vx, g, s, m), x, g.nx, true, tx);
        staps<LU, W>(P.vs, g, s, m, x, true, P.order, ts);
        vec<LS, W> div = OS::add(fold<LS, LU, W>(c, tx, P.order), fold<LS, LU, W>(c, ts, P.order));
        if (P.d3) {
            mtaps<LU, W>(P.vm, g, s, m, x, true, P.order, tm);
            div = OS::add(div, fold<LS, LU, W>(c, tm, P.order));
        }
        int src_lane = -1;
        if (P.has_src && s == P.src_s && m == P.src_m && P.src_x >= x && P.src_x < x + W)
            src_lane = (int)(P.src_x - x);
        const vec<LU, W> p_old = vload<LU, W>(frow<TU>(P.p, g, s, m) + x);
        vec<LU, W> u = p_old;
        vec<LU, W> rr = comp ? vload<LU, W>(frow<TU>(P.rp, g, s, m) + x) : vec<LU, W>{};
        finish<LS, LU, W>(div, &P.beta, s, m, x, dt, P.variant, src_lane, src, u, rr);
        store_field<LU, W>(P.p, g, s, m, x, u);
        if (!vfinite<LU, W>(u)) mask |= 1u << P.p.bit;
        if (comp) {
            store_field<LU, W>(P.rp, g, s, m, x, rr);
            if (!vfinite<LU, W>(rr)) mask |= 1u << P.rp.bit;
        }
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
__global__ void __launch_bounds__(BLOCK) k_ac_energy(AcParams P) {
    using TU = typename lane<LU>::T;
    const Geom& g = P.g;
    const int64_t nxv = g.nx / W;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (xv < nxv && s < P.p.rows) {
        const int64_t x = xv * W;
        vec<LU, W> p = vload<LU, W>(frow<TU>(P.p, g, s, m) + x);
        vec<LU, W> vx = vload<LU, W>(frow<TU>(P.vx, g, s, m) + x);
        vec<LU, W> vs = vload<LU, W>(frow<TU>(P.vs, g, s, m) + x);
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
            vec<LU, W> vm = vload<LU, W>(frow<TU>(P.vm, g, s, m) + x);
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
