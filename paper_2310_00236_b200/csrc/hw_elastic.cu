// hw_elastic.cu — elastic velocity-stress leapfrog phase kernels (sm_100a).
//
// Per step n (ElasticSolver._step_work, elastic.py:176-238):
//   velocity phase: vx, v_slow (+ source at n dt), v_mid from sigma^n  -> k_el_vel
//   stress phase:   sxx, s_slow, s_mid, shear stresses from v^{n+1/2}  -> k_el_stress
//                   (+ fused fp64 energy partials, diagnostics.py:100-162)
// Free surfaces (2D, slow axis) come in through the ghost slabs: odd images for
// sxy/syy, even images for vx/vy (stencil.py:121-159); the surface rows of sxx use
// the plane-stress modulus and syy takes a zero increment (elastic.py:215-230).
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

template <int LU, int W>
__device__ __forceinline__ vec<LU, W> ld(const FieldView& f, const Cell& c) {
    return vload<LU, W>(fptr<typename lane<LU>::T>(f, c));
}

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK, 8) k_el_vel(ElParams P, int64_t n, double src) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    using OS = vops<LS, W>;
    const Geom& g = P.g;
    const int64_t nxv = g.nx / W;
    const int64_t rows = P.vx.rows > P.vs.rows ? P.vx.rows : P.vs.rows;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    unsigned int mask = 0;
    if (xv < nxv && s < rows) {
        const int64_t x = xv * W;
        const Cell cl = make_cell(g, s, m, x);
        TS c[4];
#pragma unroll
        for (int j = 0; j < 4; j++) c[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        vec<LU, W> t[4];
        if (s < P.vx.rows) {  // vx: fl(fl(ddx sxx + dds sxy) + ddm sxm) / rho_x (elastic.py:191-194)
            xtaps_c<LU, W>(fptr<TU>(P.sxx, cl), cl, false, t);
            vec<LS, W> a = fold<LS, LU, W>(c, t, P.order);
            staps_c<LU, W>(fptr<TU>(P.sxs, cl), cl, true, P.order, t);
            a = OS::add(a, fold<LS, LU, W>(c, t, P.order));
            if (P.d3) {
                mtaps_c<LU, W>(fptr<TU>(P.sxm, cl), cl, true, P.order, t);
                a = OS::add(a, fold<LS, LU, W>(c, t, P.order));
            }
            vec<LU, W> u = ld<LU, W>(P.vx, cl);
            vec<LU, W> rr = comp ? ld<LU, W>(P.rvx, cl) : vec<LU, W>{};
            finish<LS, LU, W>(a, &P.rho_x, s, m, x, dt, P.variant, -1, 0.0, u, rr);
            upd_store<LU, W>(P.vx, P.rvx, cl, s, u, rr, comp, mask);
        }
        if (s < P.vs.rows) {  // vy: fl(fl(ddx sxy + dds syy) + ddm sms) (+ src) / rho_y (elastic.py:196-205)
            xtaps_c<LU, W>(fptr<TU>(P.sxs, cl), cl, true, t);
            vec<LS, W> a = fold<LS, LU, W>(c, t, P.order);
            staps_c<LU, W>(fptr<TU>(P.sss, cl), cl, false, P.order, t);
            a = OS::add(a, fold<LS, LU, W>(c, t, P.order));
            if (P.d3) {
                mtaps_c<LU, W>(fptr<TU>(P.sms, cl), cl, true, P.order, t);
                a = OS::add(a, fold<LS, LU, W>(c, t, P.order));
            }
            int src_lane = -1;
            if (P.src_kind == 2 && s == P.src_s && m == P.src_m && P.src_x >= x && P.src_x < x + W)
                src_lane = (int)(P.src_x - x);
            vec<LU, W> u = ld<LU, W>(P.vs, cl);
            vec<LU, W> rr = comp ? ld<LU, W>(P.rvs, cl) : vec<LU, W>{};
            finish<LS, LU, W>(a, &P.rho_s, s, m, x, dt, P.variant, src_lane, src, u, rr);
            upd_store<LU, W>(P.vs, P.rvs, cl, s, u, rr, comp, mask);
            if (P.d3) {  // v_mid: fl(fl(ddx sxm + dds sms) + ddm smm) / rho_m
                xtaps_c<LU, W>(fptr<TU>(P.sxm, cl), cl, true, t);
                vec<LS, W> b = fold<LS, LU, W>(c, t, P.order);
                staps_c<LU, W>(fptr<TU>(P.sms, cl), cl, true, P.order, t);
                b = OS::add(b, fold<LS, LU, W>(c, t, P.order));
                mtaps_c<LU, W>(fptr<TU>(P.smm, cl), cl, false, P.order, t);
                b = OS::add(b, fold<LS, LU, W>(c, t, P.order));
                vec<LU, W> um = ld<LU, W>(P.vm, cl);
                vec<LU, W> rm = comp ? ld<LU, W>(P.rvm, cl) : vec<LU, W>{};
                finish<LS, LU, W>(b, &P.rho_m, s, m, x, dt, P.variant, -1, 0.0, um, rm);
                upd_store<LU, W>(P.vm, P.rvm, cl, s, um, rm, comp, mask);
            }
        }
    }
    record_failure(P.ctrl, n, mask);
}

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK, 8) k_el_stress(ElParams P, int64_t n, double src, int sample) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    using OS = vops<LS, W>;
    const Geom& g = P.g;
    const int64_t nxv = g.nx / W;
    const int64_t rows = P.sxx.rows > P.sxs.rows ? P.sxx.rows : P.sxs.rows;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    unsigned int mask = 0;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (xv < nxv && s < rows) {
        const int64_t x = xv * W;
        const Cell cl = make_cell(g, s, m, x);
        TS c[4];
#pragma unroll
        for (int j = 0; j < 4; j++) c[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        vec<LU, W> t[4], vxt[4], vst[4], vmt[4];
        if (s < P.sxx.rows) {
            xtaps_c<LU, W>(fptr<TU>(P.vx, cl), cl, true, vxt);
            vec<LS, W> dvx = fold<LS, LU, W>(c, vxt, P.order);
            vec<LS, W> dvs{}, dvm{};
            const int64_t sg = P.sxx.row0 + s;  // global row: free surfaces are global rows 0 and ns
            const bool surf = P.fs && (sg == 0 || sg == P.sxx.nglob - 1);
            if (!surf || s < P.vs.rows) {
                staps_c<LU, W>(fptr<TU>(P.vs, cl), cl, true, P.order, vst);
                dvs = fold<LS, LU, W>(c, vst, P.order);
            }
            if (P.d3) {
                mtaps_c<LU, W>(fptr<TU>(P.vm, cl), cl, true, P.order, vmt);
                dvm = fold<LS, LU, W>(c, vmt, P.order);
            }
            const vec<LS, W> stiff = pload<LS, W>(P.stiff, s, m, x);
            const vec<LS, W> lam = pload<LS, W>(P.lam, s, m, x);
            int src_lane = -1;
            if (P.src_kind == 3 && s == P.src_s && m == P.src_m && P.src_x >= x && P.src_x < x + W)
                src_lane = (int)(P.src_x - x);
            // sxx: fl(fl(stiff dvx) + fl(lam dvs)) [+ fl(lam dvm)]; surface rows fl(ep dvx) (elastic.py:215-221)
            vec<LS, W> a;
            if (surf) {
                a = OS::mul(pload<LS, W>(P.ep, sg == 0 ? 0 : 1, 0, x), dvx);
            } else {
                a = OS::add(OS::mul(stiff, dvx), OS::mul(lam, dvs));
                if (P.d3) a = OS::add(a, OS::mul(lam, dvm));
            }
            const vec<LU, W> sxx_old = ld<LU, W>(P.sxx, cl);
            vec<LU, W> u = sxx_old;
            vec<LU, W> rr = comp ? ld<LU, W>(P.rsxx, cl) : vec<LU, W>{};
            finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, src_lane, src, u, rr);
            upd_store<LU, W>(P.sxx, P.rsxx, cl, s, u, rr, comp, mask);
            const vec<LU, W> sxx_new = u;
            // s_slow: fl(fl(lam dvx) + fl(stiff dvs)) [+ fl(lam dvm)]; surface rows: zero increment (elastic.py:223-230)
            if (surf) {
                a = vsplat<LS, W>(lane<LS>::zero());
            } else {
                a = OS::add(OS::mul(lam, dvx), OS::mul(stiff, dvs));
                if (P.d3) a = OS::add(a, OS::mul(lam, dvm));
            }
            const vec<LU, W> sss_old = ld<LU, W>(P.sss, cl);
            u = sss_old;
            rr = comp ? ld<LU, W>(P.rsss, cl) : vec<LU, W>{};
            finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, src_lane, src, u, rr);
            upd_store<LU, W>(P.sss, P.rsss, cl, s, u, rr, comp, mask);
            const vec<LU, W> sss_new = u;
            vec<LU, W> smm_old{}, smm_new{};
            if (P.d3) {  // s_mid: fl(fl(fl(lam dvx) + fl(lam dvs)) + fl(stiff dvm))
                a = OS::add(OS::add(OS::mul(lam, dvx), OS::mul(lam, dvs)), OS::mul(stiff, dvm));
                smm_old = ld<LU, W>(P.smm, cl);
                u = smm_old;
                rr = comp ? ld<LU, W>(P.rsmm, cl) : vec<LU, W>{};
                finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, src_lane, src, u, rr);
                upd_store<LU, W>(P.smm, P.rsmm, cl, s, u, rr, comp, mask);
                smm_new = u;
            }
            if (sample) {  // kinetic x + strain energy at this integer-slow row (diagnostics.py:100-162)
                const double w = surf ? 0.5 : 1.0;
#pragma unroll
                for (int i = 0; i < W; i++) {
                    const int64_t xi = x + i;
                    double v = lane<LU>::to_f64(vxt[2].e[i]);
                    e[0] += (w * p64(P.e_rho_x, s, m, xi)) * (v * v);
                    double lamd = p64(P.e_lam, s, m, xi), mu = p64(P.e_mu, s, m, xi);
                    double xn = lane<LU>::to_f64(sxx_old.e[i]), x1 = lane<LU>::to_f64(sxx_new.e[i]);
                    double sn = lane<LU>::to_f64(sss_old.e[i]), s1 = lane<LU>::to_f64(sss_new.e[i]);
                    double stiffd = lamd + 2.0 * mu;
                    double dd = 4.0 * mu * (lamd + mu);
                    double val;
                    if (!P.d3) {
                        if (mu == 0.0) val = surf ? 0.0 : (xn * x1) / (lamd + mu);
                        else if (surf) val = xn * x1 * stiffd / dd;
                        else val = (stiffd * (xn * x1 + sn * s1) - lamd * (xn * s1 + sn * x1)) / dd;
                        if (surf) val = 0.5 * val;
                    } else {
                        if (mu == 0.0) {
                            val = (xn * x1) / (lamd + mu);
                        } else {
                            double mn = lane<LU>::to_f64(smm_old.e[i]), m1 = lane<LU>::to_f64(smm_new.e[i]);
                            double trn = xn + sn + mn, tr1 = x1 + s1 + m1;
                            double dot = xn * x1 + sn * s1 + mn * m1;
                            val = dot / (2.0 * mu) - lamd * trn * tr1 / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                        }
                    }
                    e[3] += val;
                    if (P.d3) {
                        double vm = lane<LU>::to_f64(vmt[2].e[i]);
                        e[2] += p64(P.e_rho_m, s, m, xi) * (vm * vm);
                    }
                }
            }
        }
        if (s < P.sxs.rows) {
            const vec<LS, W> mu = pload<LS, W>(P.mu_n, s, m, x);
            // sxy: fl(mu fl(dds vx + ddx vy)) (elastic.py:232-238)
            staps_c<LU, W>(fptr<TU>(P.vx, cl), cl, false, P.order, t);
            vec<LS, W> a = fold<LS, LU, W>(c, t, P.order);
            xtaps_c<LU, W>(fptr<TU>(P.vs, cl), cl, false, vst);
            a = OS::mul(mu, OS::add(a, fold<LS, LU, W>(c, vst, P.order)));
            vec<LU, W> old[3], nw[3];
            old[0] = ld<LU, W>(P.sxs, cl);
            vec<LU, W> u = old[0];
            vec<LU, W> rr = comp ? ld<LU, W>(P.rsxs, cl) : vec<LU, W>{};
            finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, -1, 0.0, u, rr);
            upd_store<LU, W>(P.sxs, P.rsxs, cl, s, u, rr, comp, mask);
            nw[0] = u;
            if (P.d3) {
                // s_xm: fl(mu fl(ddm vx + ddx vm))
                mtaps_c<LU, W>(fptr<TU>(P.vx, cl), cl, false, P.order, t);
                a = fold<LS, LU, W>(c, t, P.order);
                xtaps_c<LU, W>(fptr<TU>(P.vm, cl), cl, false, t);
                a = OS::mul(mu, OS::add(a, fold<LS, LU, W>(c, t, P.order)));
                old[1] = ld<LU, W>(P.sxm, cl);
                u = old[1];
                rr = comp ? ld<LU, W>(P.rsxm, cl) : vec<LU, W>{};
                finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, -1, 0.0, u, rr);
                upd_store<LU, W>(P.sxm, P.rsxm, cl, s, u, rr, comp, mask);
                nw[1] = u;
                // s_ms: fl(mu fl(dds vm + ddm vs))
                staps_c<LU, W>(fptr<TU>(P.vm, cl), cl, false, P.order, t);
                a = fold<LS, LU, W>(c, t, P.order);
                mtaps_c<LU, W>(fptr<TU>(P.vs, cl), cl, false, P.order, t);
                a = OS::mul(mu, OS::add(a, fold<LS, LU, W>(c, t, P.order)));
                old[2] = ld<LU, W>(P.sms, cl);
                u = old[2];
                rr = comp ? ld<LU, W>(P.rsms, cl) : vec<LU, W>{};
                finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, -1, 0.0, u, rr);
                upd_store<LU, W>(P.sms, P.rsms, cl, s, u, rr, comp, mask);
                nw[2] = u;
            }
            if (sample) {  // kinetic slow + shear energy at this half-slow row
                vec<LU, W> vsv = ld<LU, W>(P.vs, cl);
                const int nsh = P.d3 ? 3 : 1;
#pragma unroll
                for (int i = 0; i < W; i++) {
                    const int64_t xi = x + i;
                    double v = lane<LU>::to_f64(vsv.e[i]);
                    e[1] += p64(P.e_rho_s, s, m, xi) * (v * v);
                    double mun = p64(P.e_mu_n, s, m, xi);
                    for (int q = 0; q < nsh; q++) {
                        double a0 = lane<LU>::to_f64(old[q].e[i]), a1 = lane<LU>::to_f64(nw[q].e[i]);
                        e[4] += mun > 0.0 ? (a0 * a1) / mun : 0.0;
                    }
                }
            }
        }
    }
    record_failure(P.ctrl, n, mask);
    if (sample) block_partials(e, P.partials);
}

// E(t=0): stresses paired with themselves (elastic.py:265-267).
template <int LU, int W>
__global__ void __launch_bounds__(BLOCK, 8) k_el_energy(ElParams P) {
    const Geom& g = P.g;
    const int64_t nxv = g.nx / W;
    const int64_t rows = P.sxx.rows > P.sxs.rows ? P.sxx.rows : P.sxs.rows;
    const int64_t xv = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t m = blockIdx.y, s = blockIdx.z;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (xv < nxv && s < rows) {
        const int64_t x = xv * W;
        const Cell cl = make_cell(g, s, m, x);
        if (s < P.sxx.rows) {
            const int64_t sg = P.sxx.row0 + s;
            const bool surf = P.fs && (sg == 0 || sg == P.sxx.nglob - 1);
            const double w = surf ? 0.5 : 1.0;
            vec<LU, W> vx = ld<LU, W>(P.vx, cl), sxx = ld<LU, W>(P.sxx, cl),
                       sss = ld<LU, W>(P.sss, cl);
            vec<LU, W> smm = P.d3 ? ld<LU, W>(P.smm, cl) : vec<LU, W>{};
            vec<LU, W> vm = P.d3 ? ld<LU, W>(P.vm, cl) : vec<LU, W>{};
#pragma unroll
            for (int i = 0; i < W; i++) {
                const int64_t xi = x + i;
                double v = lane<LU>::to_f64(vx.e[i]);
                e[0] += (w * p64(P.e_rho_x, s, m, xi)) * (v * v);
                double lamd = p64(P.e_lam, s, m, xi), mu = p64(P.e_mu, s, m, xi);
                double xn = lane<LU>::to_f64(sxx.e[i]), sn = lane<LU>::to_f64(sss.e[i]);
                double stiffd = lamd + 2.0 * mu;
                double dd = 4.0 * mu * (lamd + mu);
                double val;
                if (!P.d3) {
                    if (mu == 0.0) val = surf ? 0.0 : (xn * xn) / (lamd + mu);
                    else if (surf) val = xn * xn * stiffd / dd;
                    else val = (stiffd * (xn * xn + sn * sn) - lamd * (xn * sn + sn * xn)) / dd;
                    if (surf) val = 0.5 * val;
                } else {
                    if (mu == 0.0) {
                        val = (xn * xn) / (lamd + mu);
                    } else {
                        double mn = lane<LU>::to_f64(smm.e[i]);
                        double tr = xn + sn + mn;
                        double dot = xn * xn + sn * sn + mn * mn;
                        val = dot / (2.0 * mu) - lamd * tr * tr / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                    }
                    double vmv = lane<LU>::to_f64(vm.e[i]);
                    e[2] += p64(P.e_rho_m, s, m, xi) * (vmv * vmv);
                }
                e[3] += val;
            }
        }
        if (s < P.sxs.rows) {
            vec<LU, W> vs = ld<LU, W>(P.vs, cl);
            vec<LU, W> sh[3];
            sh[0] = ld<LU, W>(P.sxs, cl);
            if (P.d3) {
                sh[1] = ld<LU, W>(P.sxm, cl);
                sh[2] = ld<LU, W>(P.sms, cl);
            }
            const int nsh = P.d3 ? 3 : 1;
#pragma unroll
            for (int i = 0; i < W; i++) {
                const int64_t xi = x + i;
                double v = lane<LU>::to_f64(vs.e[i]);
                e[1] += p64(P.e_rho_s, s, m, xi) * (v * v);
                double mun = p64(P.e_mu_n, s, m, xi);
                for (int q = 0; q < nsh; q++) {
                    double a0 = lane<LU>::to_f64(sh[q].e[i]);
                    e[4] += mun > 0.0 ? (a0 * a0) / mun : 0.0;
                }
            }
        }
    }
    block_partials(e, P.partials);
}

void launch_el_vel(int LS, int LU, int W, const ElParams& P, int64_t n, double src, int64_t nblocks, cudaStream_t st) {
    HW_DISPATCH_LS(LS, HW_DISPATCH_LU(LU, HW_DISPATCH_W(W, k_el_vel<LS_, LU_, W_><<<grid3(P.g, W, nblocks), block3(P.g, W), 0, st>>>(P, n, src))))
}
void launch_el_stress(int LS, int LU, int W, const ElParams& P, int64_t n, double src, int sample, int64_t nblocks,
                      cudaStream_t st) {
    HW_DISPATCH_LS(LS, HW_DISPATCH_LU(LU, HW_DISPATCH_W(W, k_el_stress<LS_, LU_, W_><<<grid3(P.g, W, nblocks), block3(P.g, W), 0, st>>>(P, n, src, sample))))
}
void launch_el_energy(int LU, int W, const ElParams& P, int64_t nblocks, cudaStream_t st) {
    HW_DISPATCH_LU(LU, HW_DISPATCH_W(W, k_el_energy<LU_, W_><<<grid3(P.g, W, nblocks), block3(P.g, W), 0, st>>>(P)))
}

}  // namespace hw
