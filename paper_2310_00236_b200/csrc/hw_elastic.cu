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
__global__ void __launch_bounds__(BLOCK) k_el_vel(ElParams P, int64_t n, double src) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    using OS = vops<LS, W>;
    const Geom& g = P.g;
    const int64_t rows = P.vx.rows > P.vs.rows ? P.vx.rows : P.vs.rows;
    const int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
    const int64_t m = blockIdx.y, s0 = (int64_t)blockIdx.z * RS;
    unsigned int mask = 0;
    if (x < g.nx && s0 < rows) {
        const int64_t s1 = s0 + RS < rows ? s0 + RS : rows;
        Cell c = make_cell(g, s0, m, x);
        TS k[4];
#pragma unroll
        for (int j = 0; j < 4; j++) k[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        Q4<LU, W> xsq, ssq, msq;  // sxy rows s-2..s+1, syy rows s-1..s+2, s_ms rows s-2..s+1
        {
            const TU* a = fptr<TU>(P.sxs, c);
            const TU* b = fptr<TU>(P.sss, c);
            xsq.q[1] = vload<LU, W>(a - 2 * c.slab); xsq.q[2] = vload<LU, W>(a - c.slab); xsq.q[3] = vload<LU, W>(a);
            ssq.q[1] = vload<LU, W>(b - c.slab); ssq.q[2] = vload<LU, W>(b); ssq.q[3] = vload<LU, W>(b + c.slab);
            if (P.d3) {
                const TU* d = fptr<TU>(P.sms, c);
                msq.q[1] = vload<LU, W>(d - 2 * c.slab); msq.q[2] = vload<LU, W>(d - c.slab); msq.q[3] = vload<LU, W>(d);
            }
        }
        #pragma unroll 1
        for (int64_t s = s0; s < s1; s++, c.off += c.slab) {
            xsq.push(vload<LU, W>(fptr<TU>(P.sxs, c) + c.slab));
            ssq.push(vload<LU, W>(fptr<TU>(P.sss, c) + 2 * c.slab));
            if (P.d3) msq.push(vload<LU, W>(fptr<TU>(P.sms, c) + c.slab));
            vec<LU, W> t[4];
            if (s < P.vx.rows) {  // vx: fl(fl(ddx sxx + dds sxy) + ddm sxm) / rho_x (elastic.py:191-194)
                xtaps_c<LU, W>(fptr<TU>(P.sxx, c), c, false, t);
                vec<LS, W> a = OS::add(fold<LS, LU, W>(k, t, P.order), fold<LS, LU, W>(k, xsq.q, P.order));
                if (P.d3) {
                    mtaps_c<LU, W>(fptr<TU>(P.sxm, c), c, true, P.order, t);
                    a = OS::add(a, fold<LS, LU, W>(k, t, P.order));
                }
                vec<LU, W> u = ld<LU, W>(P.vx, c);
                vec<LU, W> rr = comp ? ld<LU, W>(P.rvx, c) : vec<LU, W>{};
                finish<LS, LU, W>(a, &P.rho_x, s, m, x, dt, P.variant, -1, 0.0, u, rr);
                upd_store<LU, W>(P.vx, P.rvx, c, s, u, rr, comp, mask);
            }
            if (s < P.vs.rows) {  // vy: fl(fl(ddx sxy + dds syy) + ddm sms) (+ src) / rho_y (elastic.py:196-205)
                xtaps_own<LU, W>(fptr<TU>(P.sxs, c), c, xsq.q[2], true, t);
                vec<LS, W> a = OS::add(fold<LS, LU, W>(k, t, P.order), fold<LS, LU, W>(k, ssq.q, P.order));
                if (P.d3) {
                    mtaps_c<LU, W>(fptr<TU>(P.sms, c), c, true, P.order, t);
                    a = OS::add(a, fold<LS, LU, W>(k, t, P.order));
                }
                int src_lane = -1;
                if (P.src_kind == 2 && s == P.src_s && m == P.src_m && P.src_x >= x && P.src_x < x + W)
                    src_lane = (int)(P.src_x - x);
                vec<LU, W> u = ld<LU, W>(P.vs, c);
                vec<LU, W> rr = comp ? ld<LU, W>(P.rvs, c) : vec<LU, W>{};
                finish<LS, LU, W>(a, &P.rho_s, s, m, x, dt, P.variant, src_lane, src, u, rr);
                upd_store<LU, W>(P.vs, P.rvs, c, s, u, rr, comp, mask);
                if (P.d3) {  // v_mid: fl(fl(ddx sxm + dds sms) + ddm smm) / rho_m
                    xtaps_c<LU, W>(fptr<TU>(P.sxm, c), c, true, t);
                    vec<LS, W> b = OS::add(fold<LS, LU, W>(k, t, P.order), fold<LS, LU, W>(k, msq.q, P.order));
                    mtaps_c<LU, W>(fptr<TU>(P.smm, c), c, false, P.order, t);
                    b = OS::add(b, fold<LS, LU, W>(k, t, P.order));
                    vec<LU, W> um = ld<LU, W>(P.vm, c);
                    vec<LU, W> rm = comp ? ld<LU, W>(P.rvm, c) : vec<LU, W>{};
                    finish<LS, LU, W>(b, &P.rho_m, s, m, x, dt, P.variant, -1, 0.0, um, rm);
                    upd_store<LU, W>(P.vm, P.rvm, c, s, um, rm, comp, mask);
                }
            }
        }
    }
    record_failure(P.ctrl, n, mask);
}

template <int LS, int LU, int W>
__global__ void __launch_bounds__(BLOCK) k_el_stress(ElParams P, int64_t n, double src, int sample) {
    if (halted(P.ctrl, n)) return;
    using TU = typename lane<LU>::T;
    using TS = typename lane<LS>::T;
    using OS = vops<LS, W>;
    const Geom& g = P.g;
    const int64_t rows = P.sxx.rows > P.sxs.rows ? P.sxx.rows : P.sxs.rows;
    const int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
    const int64_t m = blockIdx.y, s0 = (int64_t)blockIdx.z * RS;
    unsigned int mask = 0;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (x < g.nx && s0 < rows) {
        const int64_t s1 = s0 + RS < rows ? s0 + RS : rows;
        Cell c = make_cell(g, s0, m, x);
        TS k[4];
#pragma unroll
        for (int j = 0; j < 4; j++) k[j] = lconst<LS>(P.k, j);
        const TU dt = lconst<LU>(P.k, 4);
        const bool comp = P.variant != 0;
        Q4<LU, W> vsq, vxq, vmq;  // vy rows s-2..s+1; vx rows s-1..s+2; v_mid rows s-1..s+2
        {
            const TU* a = fptr<TU>(P.vs, c);
            const TU* b = fptr<TU>(P.vx, c);
            vsq.q[1] = vload<LU, W>(a - 2 * c.slab); vsq.q[2] = vload<LU, W>(a - c.slab); vsq.q[3] = vload<LU, W>(a);
            vxq.q[1] = vload<LU, W>(b - c.slab); vxq.q[2] = vload<LU, W>(b); vxq.q[3] = vload<LU, W>(b + c.slab);
            if (P.d3) {
                const TU* d = fptr<TU>(P.vm, c);
                vmq.q[1] = vload<LU, W>(d - c.slab); vmq.q[2] = vload<LU, W>(d); vmq.q[3] = vload<LU, W>(d + c.slab);
            }
        }
        #pragma unroll 1
        for (int64_t s = s0; s < s1; s++, c.off += c.slab) {
            vsq.push(vload<LU, W>(fptr<TU>(P.vs, c) + c.slab));
            vxq.push(vload<LU, W>(fptr<TU>(P.vx, c) + 2 * c.slab));
            if (P.d3) vmq.push(vload<LU, W>(fptr<TU>(P.vm, c) + 2 * c.slab));
            vec<LU, W> t[4], vxt[4];
            if (s < P.sxx.rows) {
                xtaps_own<LU, W>(fptr<TU>(P.vx, c), c, vxq.q[1], true, vxt);
                vec<LS, W> dvx = fold<LS, LU, W>(k, vxt, P.order);
                vec<LS, W> dvs = fold<LS, LU, W>(k, vsq.q, P.order);
                vec<LS, W> dvm{};
                if (P.d3) {
                    mtaps_c<LU, W>(fptr<TU>(P.vm, c), c, true, P.order, t);
                    dvm = fold<LS, LU, W>(k, t, P.order);
                }
                const int64_t sg = P.sxx.row0 + s;  // global row: free surfaces are global rows 0 and ns
                const bool surf = P.fs && (sg == 0 || sg == P.sxx.nglob - 1);
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
                const vec<LU, W> sxx_old = ld<LU, W>(P.sxx, c);
                vec<LU, W> u = sxx_old;
                vec<LU, W> rr = comp ? ld<LU, W>(P.rsxx, c) : vec<LU, W>{};
                finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, src_lane, src, u, rr);
                upd_store<LU, W>(P.sxx, P.rsxx, c, s, u, rr, comp, mask);
                const vec<LU, W> sxx_new = u;
                // s_slow: fl(fl(lam dvx) + fl(stiff dvs)) [+ fl(lam dvm)]; surface rows: zero increment (elastic.py:223-230)
                if (surf) {
                    a = vsplat<LS, W>(lane<LS>::zero());
                } else {
                    a = OS::add(OS::mul(lam, dvx), OS::mul(stiff, dvs));
                    if (P.d3) a = OS::add(a, OS::mul(lam, dvm));
                }
                const vec<LU, W> sss_old = ld<LU, W>(P.sss, c);
                u = sss_old;
                rr = comp ? ld<LU, W>(P.rsss, c) : vec<LU, W>{};
                finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, src_lane, src, u, rr);
                upd_store<LU, W>(P.sss, P.rsss, c, s, u, rr, comp, mask);
                const vec<LU, W> sss_new = u;
                vec<LU, W> smm_old{}, smm_new{};
                if (P.d3) {  // s_mid: fl(fl(fl(lam dvx) + fl(lam dvs)) + fl(stiff dvm))
                    a = OS::add(OS::add(OS::mul(lam, dvx), OS::mul(lam, dvs)), OS::mul(stiff, dvm));
                    smm_old = ld<LU, W>(P.smm, c);
                    u = smm_old;
                    rr = comp ? ld<LU, W>(P.rsmm, c) : vec<LU, W>{};
                    finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, src_lane, src, u, rr);
                    upd_store<LU, W>(P.smm, P.rsmm, c, s, u, rr, comp, mask);
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
                        double sn = lane<LU>::to_f64(sss_old.e[i]), s1v = lane<LU>::to_f64(sss_new.e[i]);
                        double stiffd = lamd + 2.0 * mu;
                        double dd = 4.0 * mu * (lamd + mu);
                        double val;
                        if (!P.d3) {
                            if (mu == 0.0) val = surf ? 0.0 : (xn * x1) / (lamd + mu);
                            else if (surf) val = xn * x1 * stiffd / dd;
                            else val = (stiffd * (xn * x1 + sn * s1v) - lamd * (xn * s1v + sn * x1)) / dd;
                            if (surf) val = 0.5 * val;
                        } else {
                            if (mu == 0.0) {
                                val = (xn * x1) / (lamd + mu);
                            } else {
                                double mn = lane<LU>::to_f64(smm_old.e[i]), m1 = lane<LU>::to_f64(smm_new.e[i]);
                                double trn = xn + sn + mn, tr1 = x1 + s1v + m1;
                                double dot = xn * x1 + sn * s1v + mn * m1;
                                val = dot / (2.0 * mu) - lamd * trn * tr1 / (2.0 * mu * (3.0 * lamd + 2.0 * mu));
                            }
                            double vm = lane<LU>::to_f64(vmq.q[1].e[i]);
                            e[2] += p64(P.e_rho_m, s, m, xi) * (vm * vm);
                        }
                        e[3] += val;
                    }
                }
            }
            if (s < P.sxs.rows) {
                const vec<LS, W> mu = pload<LS, W>(P.mu_n, s, m, x);
                // sxy: fl(mu fl(dds vx + ddx vy)) (elastic.py:232-238)
                vec<LS, W> a = fold<LS, LU, W>(k, vxq.q, P.order);
                xtaps_own<LU, W>(fptr<TU>(P.vs, c), c, vsq.q[2], false, t);
                a = OS::mul(mu, OS::add(a, fold<LS, LU, W>(k, t, P.order)));
                vec<LU, W> old[3], nw[3];
                old[0] = ld<LU, W>(P.sxs, c);
                vec<LU, W> u = old[0];
                vec<LU, W> rr = comp ? ld<LU, W>(P.rsxs, c) : vec<LU, W>{};
                finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, -1, 0.0, u, rr);
                upd_store<LU, W>(P.sxs, P.rsxs, c, s, u, rr, comp, mask);
                nw[0] = u;
                if (P.d3) {
                    // s_xm: fl(mu fl(ddm vx + ddx vm))
                    mtaps_c<LU, W>(fptr<TU>(P.vx, c), c, false, P.order, t);
                    a = fold<LS, LU, W>(k, t, P.order);
                    xtaps_own<LU, W>(fptr<TU>(P.vm, c), c, vmq.q[1], false, t);
                    a = OS::mul(mu, OS::add(a, fold<LS, LU, W>(k, t, P.order)));
                    old[1] = ld<LU, W>(P.sxm, c);
                    u = old[1];
                    rr = comp ? ld<LU, W>(P.rsxm, c) : vec<LU, W>{};
                    finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, -1, 0.0, u, rr);
                    upd_store<LU, W>(P.sxm, P.rsxm, c, s, u, rr, comp, mask);
                    nw[1] = u;
                    // s_ms: fl(mu fl(dds vm + ddm vs))
                    a = fold<LS, LU, W>(k, vmq.q, P.order);
                    mtaps_c<LU, W>(fptr<TU>(P.vs, c), c, false, P.order, t);
                    a = OS::mul(mu, OS::add(a, fold<LS, LU, W>(k, t, P.order)));
                    old[2] = ld<LU, W>(P.sms, c);
                    u = old[2];
                    rr = comp ? ld<LU, W>(P.rsms, c) : vec<LU, W>{};
                    finish<LS, LU, W>(a, nullptr, s, m, x, dt, P.variant, -1, 0.0, u, rr);
                    upd_store<LU, W>(P.sms, P.rsms, c, s, u, rr, comp, mask);
                    nw[2] = u;
                }
                if (sample) {  // kinetic slow + shear energy at this half-slow row
                    const vec<LU, W> vsv = vsq.q[2];
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
    }
    record_failure(P.ctrl, n, mask);
    if (sample) block_partials(e, P.partials);
}

// E(t=0): stresses paired with themselves (elastic.py:265-267).
template <int LU, int W>
__global__ void __launch_bounds__(BLOCK) k_el_energy(ElParams P) {
    const Geom& g = P.g;
    const int64_t rows = P.sxx.rows > P.sxs.rows ? P.sxx.rows : P.sxs.rows;
    const int64_t x = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * W;
    const int64_t m = blockIdx.y, s0 = (int64_t)blockIdx.z * RS;
    double e[NCOMP] = {0.0, 0.0, 0.0, 0.0, 0.0};
    if (x < g.nx && s0 < rows) {
        const int64_t s1 = s0 + RS < rows ? s0 + RS : rows;
        Cell cl = make_cell(g, s0, m, x);
        #pragma unroll 1
        for (int64_t s = s0; s < s1; s++, cl.off += cl.slab) {
            if (s < P.sxx.rows) {
                const int64_t sg = P.sxx.row0 + s;
                const bool surf = P.fs && (sg == 0 || sg == P.sxx.nglob - 1);
                const double w = surf ? 0.5 : 1.0;
                vec<LU, W> vx = ld<LU, W>(P.vx, cl), sxx = ld<LU, W>(P.sxx, cl), sss = ld<LU, W>(P.sss, cl);
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
