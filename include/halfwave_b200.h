/*
 * halfwave_b200.h — C ABI of the B200 (sm_100a) staggered-grid leapfrog hot path.
 *
 * This is the drop-in boundary for the reference package's solver entry points
 * (reference: /root/reference/pkg/src/halfwave, "halfwave"):
 *
 *   AcousticSolver.__init__ / .run / .step_baseline / .step_compensated
 *       acoustic.py:56-97, 113-128, 185-236
 *   ElasticSolver.__init__ / .run / .step_baseline / .step_compensated
 *       elastic.py:63-113, 132-147, 242-296
 *
 * The reference has no FFI of its own (pure Python/numpy); these entry points are
 * what its Python classes would bind with ctypes, one call per run()/step_*().
 * The whole `for n in range(nt)` loop (acoustic.py:210-226, elastic.py:271-286)
 * runs behind hw_run(); the host crosses the boundary once per call.
 *
 * Plain C types only: pointers, sizes, fixed-width integers, IEEE doubles.
 * No C++ exceptions cross this boundary; every entry point returns an hw_status.
 *
 * Axis naming is generic so one descriptor covers 2D and 3D:
 *   x   — fastest axis (reference 2D "x", periodic)
 *   mid — 3D only (3D "y"); nm == 1 in 2D
 *   slow— slab / slowest axis (reference 2D "y", 3D "z"); free surfaces live here
 * Arrays are row-major with x fastest ([s][m][x]), matching grids.py:3.
 */
#ifndef HALFWAVE_B200_H
#define HALFWAVE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HW_ABI_VERSION 1

typedef enum hw_status {
    HW_OK = 0,
    HW_RANGE_FAILURE = 1, /* RangeFailureError (diagnostics.py:24-32); state holds the failing step */
    HW_EINVAL = 2,        /* bad argument (ValueError in the reference) */
    HW_ECUDA = 3,         /* CUDA runtime error */
    HW_ENCCL = 4          /* NCCL error (multi-GPU halo exchange) */
} hw_status;

enum hw_equation { HW_EQ_ACOUSTIC = 0, HW_EQ_ELASTIC = 1 };        /* MediumKind, grids.py:126-128 */
enum hw_lane { HW_FP16 = 16, HW_FP32 = 32, HW_FP64 = 64 };         /* Precision, precision.py:35-41 */
enum hw_variant { HW_NAIVE = 0, HW_OP3 = 3, HW_OP6 = 6 };          /* None / Variant.OP3 / OP6, efsum.py:30-37 */
enum hw_bc { HW_BC_PERIODIC = 0, HW_BC_FREE_SURFACE = 1 };         /* Boundary, grids.py:59-64 */
enum hw_source {
    HW_SRC_NONE = 0,
    HW_SRC_PRESSURE = 1,  /* SourceKind.PRESSURE_POINT, acoustic.py:176-181 */
    HW_SRC_VSLOW = 2,     /* SourceKind.VY_POINT (2D vy / 3D vz), elastic.py:196-205 */
    HW_SRC_EXPLOSIVE = 3  /* extension: into every normal-stress increment at (n+1/2) dt */
};

/* fp64 medium planes, already materialised on the host exactly as the reference
 * builds them (extend_rows grids.py:321-331; lam + 2.0*mu, elastic.py:104;
 * 4.0*mu*(lam+mu)/(lam+2.0*mu), elastic.py:110-113).  Each plane has the shape of
 * the field it feeds (noted).  The library rounds each into its lane once
 * (UpdatePipeline.update_plane / stencil_plane, stepping.py:47-56) and keeps the
 * fp64 copies for the energy functionals (diagnostics.py:76-162). */
enum hw_plane {
    HW_PL_RHO_X = 0, /* shape of vx;  acoustic + elastic; U lane */
    HW_PL_RHO_S = 1, /* shape of v_slow */
    HW_PL_RHO_M = 2, /* shape of v_mid (3D only) */
    HW_PL_BETA = 3,  /* shape of p (acoustic) */
    HW_PL_LAM = 4,   /* shape of sxx (elastic); S lane + energy */
    HW_PL_MU = 5,    /* shape of sxx (cell mu, energy only) */
    HW_PL_STIFF = 6, /* shape of sxx: lam + 2 mu; S lane */
    HW_PL_MU_N = 7,  /* shape of the shear stresses (node/edge mu reuses cell mu); S lane + energy */
    HW_PL_EP = 8,    /* [2][nx]: plane-stress modulus on the top / bottom surface rows (free surface) */
    HW_NPLANES = 9
};

typedef struct hw_desc {
    int32_t abi_version;  /* HW_ABI_VERSION */
    int32_t equation;     /* hw_equation */
    int32_t ndim;         /* 2 or 3 */
    int32_t order;        /* 4 (reference, stencil.py:34) or 2 (extension: inner tap pair only) */
    int32_t bc_slow;      /* hw_bc on the slow axis; x and mid are periodic */
    int32_t lane_s;       /* stencil precision */
    int32_t lane_u;       /* update precision */
    int32_t src_kind;     /* hw_source */
    int64_t nx, nm, ns;   /* cells along x, mid (1 in 2D), slow */
    double dx;            /* GridSpec.dx */
    double dt;            /* GridSpec.dt, raw fp64; rounded into U by the library (stepping.py:30) */
    double taps[4];       /* c1..c4 of StencilSpec.make, already rounded into lane_s (stencil.py:52-56) */
    const double* plane[HW_NPLANES];
    int64_t src_x, src_m, src_s;  /* source cell on its field's sub-grid */
    const int64_t* receivers;     /* n_receivers triples (x, m, s); trace field is p (acoustic) or v_slow (elastic) */
    int32_t n_receivers;
    int32_t world_size;           /* slab decomposition over the slow axis; 1 = single GPU */
    int32_t rank;
    int32_t device;               /* CUDA device ordinal for this rank */
    const void* nccl_unique_id;   /* 128-byte ncclUniqueId when world_size > 1 */
    int64_t energy_every;         /* AcousticSolver(energy_every=...), >= 1 */
} hw_desc;

typedef struct hw_solver hw_solver; /* opaque; owns device state, medium, streams, NCCL comm */

/* Number of state fields (solution + residual) and their external order:
 *   acoustic 2D: p vx vy rp rvx rvy                       (AcousticState, acoustic.py:35-50)
 *   acoustic 3D: p vx vy vz rp rvx rvy rvz
 *   elastic 2D : vx vy sxx syy sxy rvx rvy rsxx rsyy rsxy (ElasticState, elastic.py:43-57)
 *   elastic 3D : vx vy vz sxx syy szz sxy sxz syz + 9 residuals
 * fail_field from hw_run indexes this list (check_finite order, acoustic.py:154-160). */
int hw_num_fields(int32_t equation, int32_t ndim);

/* Shape of external field f as (slow, mid, x) extents. */
int hw_field_shape(const hw_desc* d, int32_t field, int64_t shape[3]);

/* Validate the descriptor, allocate device state (zeros) and materialise the medium.
 * Mirrors the solver constructors (acoustic.py:56-97, elastic.py:63-113).  The host
 * side has already done the reference's ValueError validation; this re-checks the
 * invariants the kernels depend on.  The handle is bound to desc->device. */
int hw_create(const hw_desc* desc, hw_solver** out);
int hw_destroy(hw_solver* h);

/* Slab decomposition over the slow axis.  Two transports:
 *  - one process per GPU: desc->world_size > 1, desc->rank, desc->device and a
 *    128-byte ncclUniqueId (from hw_nccl_unique_id on rank 0, broadcast by the
 *    host) -> hw_create; halo slabs move by NCCL send/recv after each phase and
 *    hw_run returns the combined energy history and traces on every rank;
 *  - one process driving nslabs slabs (on one GPU or several NVLink peers):
 *    hw_create_group creates the nslabs handles (devices[r], or desc->device for
 *    all when devices is NULL) and hw_run_group marches them in lockstep with
 *    peer copies of the halo slabs.  Destroying any handle releases the group.
 * Slab r owns global slow rows [r*ns/N, (r+1)*ns/N) (+ the extra free-surface row
 * on the last slab); hw_set_state / hw_get_state take the global host arrays. */
int hw_nccl_unique_id(void* out128);

/* The halo plan both transports execute (host only, no CUDA): for slab `rank` of `world`,
 * the point-to-point transfers of one exchange in issue order.  row0 / nrows are local slow
 * rows of external field `field` (row0 < 0: top ghost rows, row0 >= local rows: bottom ghost
 * rows); peer is the rank sent to (send = 1) or received from (send = 0).  The k-th receive
 * of rank b from rank a pairs with the k-th send of a to b.  Kinds: */
enum hw_plan_kind {
    HW_PLAN_VEL = 0,    /* after the velocity phase: velocities with slow-axis derivatives */
    HW_PLAN_STRESS = 1, /* after the pressure / stress phase: the other ghosted fields */
    HW_PLAN_FUSED = 2,  /* once per step of the fused 2D acoustic kernel: p, vy, rvy (3 rows) */
    HW_PLAN_FUSED_EL3 = 3, /* once per step of the one-pass 3D elastic kernel: the six stresses (2 rows),
                            * the velocities and their residuals (1 row) */
    HW_PLAN_FUSED_AC3 = 4, /* once per step of the one-pass 3D acoustic kernels: p, v_slow, its residual (1 row) */
    HW_PLAN_FUSED_EL2 = 5  /* once per step of the one-pass 2D elastic kernel: the five fields and the velocity
                            * residuals (3 rows) */
};
typedef struct hw_xfer {
    int32_t field, peer, send, pad;
    int64_t row0, nrows;
} hw_xfer;
/* *n receives the number of transfers; at most cap are written to out (out may be NULL). */
int hw_exchange_plan(const hw_desc* desc, int32_t world, int32_t rank, int32_t kind, hw_xfer* out, int32_t cap,
                     int32_t* n);
int hw_create_group(const hw_desc* desc, int32_t nslabs, const int32_t* devices, hw_solver** out);
int hw_run_group(hw_solver* const* handles, int32_t nslabs, int32_t variant, int64_t step0, int64_t nt,
                 const double* src_samples, double* traces, double* e_times, double* e_vals,
                 int64_t* n_energy, int64_t* fail_step, int32_t* fail_field);

/* Upload / download every state field in external order.  Each pointer addresses a
 * row-major host array of lane_u storage (uint16 fp16 bits, float, or double) with
 * the field's full (global) shape; a rank > 0 of a multi-GPU job reads/writes only
 * its own slab rows.  Mirrors _load_work / _flush_work (acoustic.py:137-152). */
int hw_set_state(hw_solver* h, const void* const* fields);
int hw_get_state(hw_solver* h, void* const* fields);

/* March nt steps from step index step0 (AcousticSolver.run, acoustic.py:185-236;
 * ElasticSolver.run, elastic.py:242-296) on the device-resident state.
 *   variant     hw_variant
 *   src_samples nt fp64 samples sample_source(t_n) (sources.py:57-69), NULL if no source
 *   traces      [n_receivers][nt] fp64 receiver samples recorded after each step
 *   e_times, e_vals  capacity 1 + nt/energy_every; E(t=0) first, then every sample step
 *   n_energy    number of energy samples written
 *   fail_step, fail_field  set on HW_RANGE_FAILURE (first non-finite field in
 *               check_finite order at the first failing step; state stops after it).
 * Any of the output pointers may be NULL.  Blocks until the device is done. */
int hw_run(hw_solver* h, int32_t variant, int64_t step0, int64_t nt, const double* src_samples,
           double* traces, double* e_times, double* e_vals, int64_t* n_energy,
           int64_t* fail_step, int32_t* fail_field);

/* Device-resident timing helper for benchmarks: same as hw_run but outputs stay on
 * the device (no host copies).  Returns the device time of the marched steps in ms
 * (CUDA events on the solver's stream) through *ms. */
int hw_run_device(hw_solver* h, int32_t variant, int64_t step0, int64_t nt,
                  const double* src_samples, float* ms);

/* Kernel launches issued by the last hw_run / hw_run_device (evidence for bench.py). */
int64_t hw_last_launch_count(const hw_solver* h);

/* Which kernel family this handle's steps use (chosen at hw_create from the lanes,
 * dimension, order, grid size and transport): "small2d" (persistent small-grid 2D kernels),
 * "fused2d" (one-pass 2D acoustic, binary16), "fused2d-tb2" (opt-in two-step 2D acoustic),
 * "fused2d-el" (one-pass 2D elastic, binary16), "fused3d" (one-pass 3D acoustic, binary16),
 * "fused3d-f32" (one-pass 3D acoustic, binary32 lanes), "fused3d-el" (opt-in one-pass 3D
 * elastic), "stream2d" / "stream3d" (streaming phase kernels) or "generic" (phase kernels,
 * every lane combination).  Static string; "" for NULL. */
const char* hw_kernel_path(const hw_solver* h);

/* Halo transport of the handle: 0 single domain, 1 in-process slab group (peer copies),
 * 2 NCCL (one process per GPU).  -1 for NULL. */
int32_t hw_transport(const hw_solver* h);

/* Average duration (ms) of the dominant (fused step) kernel in the last
 * hw_run_device, measured with CUDA events on the launching stream; 0 if unknown. */
double hw_last_kernel_ms(const hw_solver* h);

/* Self-test: compare the branch-free binary16 division used for medium divisors
 * against the IEEE path (__fdiv_rn, then one RNE to binary16) for all 2^16 x
 * (2^16 - 2050) operand pairs on `device`.  *mismatches receives the count;
 * *first_pair the first failing (a << 16 | b) bit patterns. */
int hw_selftest_div16(int32_t device, uint64_t* mismatches, uint32_t* first_pair);

/* Self-test of the guarded allocations (option "guard"): allocates 4096 bytes and reads the byte at
 * `offset` from a kernel.  With guard = 1, offset -1 faults (HW_ECUDA; the CUDA context is lost, so call
 * it from a process of its own); with guard = 2, offset 4096 faults; offsets 0 .. 4095 return HW_OK. */
int hw_selftest_guard(int32_t device, int64_t offset);

/* The exhaustive per-divisor table behind the cheap binary16 division: bit b of
 * the 1024 words is set iff fl16(fl32(a * rcp_rn(b))) == fl16(a / b) for every
 * binary16 a (b = positive finite binary16 bit pattern).  Computed on `device`. */
int hw_cheap_div_table(int32_t device, uint32_t* bits1024);

/* Division mode the solver picked for a divisor plane (0 none, 1 fast exact,
 * 2 IEEE, 3 cheap table-verified); -1 on bad arguments. */
int hw_plane_div_mode(const hw_solver* h, int32_t plane);

/* Process-wide kernel-path options, read when a handle is created (no
 * environment variables are consulted).  Defaults are the production choices:
 *   "path"      0 fastest eligible kernels | 1 generic phase kernels only
 *   "div"       binary16 division: 0 per-plane choice | 1 no table path | 2 IEEE only
 *   "small"     1 persistent small-grid 2D kernels (grids <= 2^20 cells) | 0 off
 *   "tb"        0 | 1 two steps per launch, fused 2D acoustic (opt-in, measured slower)
 *   "fused_el"  1 one-pass 2D elastic kernel | 0 two-phase kernels
 *   "fused3"    1 one-pass 3D acoustic kernels | 0 two-phase kernels
 *   "fused_el3" 1 one-pass 3D elastic kernel (2nd order, media constant along x) | 0 two-phase
 *   "el3_group" 4 at most this many CTAs of the one-pass 3D elastic kernel stream adjacent tiles
 *   "ac3_group" 4 the same for the one-pass 3D acoustic kernels (binary16 and binary32)
 *   "el3_overlap_min_rows" 0 | n: NCCL slabs thinner than n slow rows run one launch and exchange in stream order
 *               (no edge / interior split; for A/B runs on a multi-GPU box)
 *   "el3_edge_ctas" 0 automatic | 1..64 CTAs of the edge launch of the one-pass 3D elastic kernel on an NCCL slab
 *   "guard"     0 | 1 | 2 every device buffer in its own mapping between unmapped pages, starting at the
 *               mapping's start (1) or ending at its end (2): out-of-bounds accesses fault (tests)
 *   "nccl_self" 0 | 1 a one-rank job given an NCCL id takes the NCCL transport (tests)
 * HW_EINVAL for an unknown name or an out-of-range value. */
int hw_set_option(const char* name, int64_t value);
int hw_get_option(const char* name, int64_t* value);

/* Thread-local message for the last non-OK status. */
const char* hw_last_error(void);

/* Library build identity (sm arch, ABI version). */
const char* hw_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HALFWAVE_B200_H */
