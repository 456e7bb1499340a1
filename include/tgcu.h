/*
 * tgcu — B200-native (sm_100a) TaylorGrid query → loss-fused backward → TV →
 * Adam hot path, behind a C ABI.
 *
 * Every entry point replaces a reference function of
 * /root/reference/proj/core (cited per declaration). Conventions:
 *   - plain pointers + sizes, no C++/torch types; all functions return an
 *     int status (TGCU_OK or one of the TGCU_ERR_* classes below, mirroring
 *     the reference's exception classes, errors.hpp:9-34) and set a
 *     thread-local message readable with tgcu_last_error();
 *   - a tgcu_grid owns the device-resident fp32 coefficients (reference AoS
 *     layout: vertex-major, x fastest, per-vertex block [f0 | f1 | f2 upper
 *     triangle], taylor_grid.hpp:27-31), the Adam moments, an optional
 *     gradient buffer and all scratch;
 *   - point/sample arrays are fp32. `flags & TGCU_HOST` means the pointers
 *     are host memory (copied in/out inside the call); otherwise device
 *     memory on the grid's device. `stream` is a cudaStream_t (NULL = the
 *     legacy default stream).
 *   - calls are synchronous (errors surface on return) unless TGCU_ASYNC is
 *     passed; async errors are sticky and reported by tgcu_sync().
 */
#ifndef TGCU_H
#define TGCU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: exception classes of errors.hpp:9-34 plus CUDA failures. */
enum {
    TGCU_OK = 0,
    TGCU_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (require_arg) */
    TGCU_ERR_CONFIG = 2,           /* tg::ConfigError */
    TGCU_ERR_INGEST = 3,           /* tg::IngestError */
    TGCU_ERR_NUMERICAL = 4,        /* tg::NumericalError */
    TGCU_ERR_RESOURCE = 5,         /* tg::ResourceError */
    TGCU_ERR_CUDA = 6              /* CUDA runtime failure / no device */
};

/* Call flags. */
enum {
    TGCU_HOST = 1,   /* point / value pointers are host memory */
    TGCU_ASYNC = 2,  /* do not synchronize; errors become sticky */
    TGCU_SORTED = 4,      /* eval: points are sorted by tgcu_sort_points (brick-binned query) */
    TGCU_EXPORT_GRAD = 8, /* train_step: also write the full gradient to the grid grad buffer
                             (validation mode; the fused path otherwise never stores it) */
    TGCU_INPUT_READY = 16, /* train_step / slab_step_begin with device samples: the caller
                             guarantees the samples are complete (no pending writes on any
                             stream), so the step's point binning need not wait for earlier
                             work on `stream` and overlaps the previous step's brick kernel */
    TGCU_HOST_RELEASE = 32 /* train_step with TGCU_HOST | TGCU_ASYNC: return once the host
                              samples have been copied (the caller may refill the buffer at
                              once); the step itself stays queued */
};

/* tg::GridSpec (grid_spec.hpp:19-24). */
typedef struct {
    int dim;           /* 2 or 3 */
    int res[3];        /* vertices per axis (>= 2); res[2] ignored for dim 2 */
    double origin[3];
    double extent[3];
    int order;         /* 0..2 */
} tgcu_grid_spec;

/* tg::InitOptions (taylor_grid.hpp:17-25). */
enum {
    TGCU_INIT_ZEROS = 0,
    TGCU_INIT_CONSTANT = 1,
    TGCU_INIT_SMALL_UNIFORM = 2,  /* reference Rng stream, host-generated (bit-identical draws) */
    TGCU_INIT_HASH_GAUSSIAN = 3   /* epsilon * N(0,1) from a counter hash of (seed, index), on
                                     device: for multi-GB throughput grids (BASELINE C4) */
};
typedef struct {
    int mode;
    double constant;
    double epsilon;
    uint64_t seed;
    uint64_t memory_cap_bytes; /* cap on fp64-equivalent coefficient bytes, as the reference */
} tgcu_init_options;

/* tg::LossConfig (sdf_loss.hpp:15-25). batch_size is the caller's n;
 * the eikonal points are the batch itself (EikonalPointSource::ReuseBatch)
 * except through tgcu_train_step_fresh_eik (FreshUniform). */
typedef struct {
    double lambda1;
    double lambda2;
    double k;
    int use_weighting;
    int use_tv;
    int differentiate_weight;
} tgcu_loss_config;

/* tg::LossTerms (schedule.hpp:43-48). */
typedef struct {
    double total;
    double fit;
    double eik;
    double tv;
} tgcu_loss_terms;

/* tg::AdamConfig (adam.hpp:9-14). */
typedef struct {
    double lr;
    double beta1;
    double beta2;
    double eps;
} tgcu_adam_config;

typedef struct tgcu_grid tgcu_grid;

const char* tgcu_last_error(void);
const char* tgcu_version(void);

/* coeff_count (grid_spec.cpp:10-19). */
int tgcu_coeff_count(int order, int dim, int* out);

/* init_grid (taylor_grid.cpp:162-188): validate (grid_spec.cpp:21-33), cap
 * check (ResourceError), allocate on `device`, initialise. opts may be NULL
 * (Zeros, 4 GiB cap). */
int tgcu_grid_create(const tgcu_grid_spec* spec, const tgcu_init_options* opts, int device,
                     tgcu_grid** out);
int tgcu_grid_destroy(tgcu_grid* g);
int tgcu_grid_spec_of(const tgcu_grid* g, tgcu_grid_spec* out);
int64_t tgcu_grid_coeff_total(const tgcu_grid* g);
/* Device pointer of the current fp32 coefficient array (AoS, coeff_total floats). */
float* tgcu_grid_coeffs(tgcu_grid* g);

/* TaylorGrid::coeffs interop in the reference layout (fp64 <-> fp32 at the boundary). */
int tgcu_grid_upload_f64(tgcu_grid* g, const double* coeffs, int64_t n);
int tgcu_grid_download_f64(tgcu_grid* g, double* coeffs, int64_t n);
int tgcu_grid_upload_f32(tgcu_grid* g, const float* coeffs, int64_t n, int flags);
int tgcu_grid_download_f32(tgcu_grid* g, float* coeffs, int64_t n, int flags);
/* all_finite (taylor_grid.cpp:190-195). */
int tgcu_grid_all_finite(tgcu_grid* g, int* out);

/* eval / eval_with_spatial_gradient (taylor_grid.cpp:197-203), batched:
 * pts n×3 (x, y, z; z ignored in 2D), values n, spatial_grad n×3 or NULL.
 * A NaN coordinate -> TGCU_ERR_INVALID_ARGUMENT (locate, grid_spec.cpp:46-48). */
int tgcu_eval(tgcu_grid* g, const float* pts, int64_t n, float* values, float* spatial_grad,
              int flags, void* stream);

/* Morton/brick sort of query points for the brick-binned query: points are
 * ordered by the Morton code of their cell's brick (8^3 / 16^2 cells), then
 * by cell inside the brick. perm (nullable) receives the source index of each
 * output point; brick_offsets (nullable, tgcu_query_brick_codes()+1 entries)
 * the start of every brick's run. Device pointers only. */
int tgcu_sort_points(tgcu_grid* g, const float* pts, int64_t n, float* sorted_pts, int64_t* perm,
                     int64_t* brick_offsets, void* stream);
int64_t tgcu_query_brick_codes(const tgcu_grid* g);
/* Brick-binned query of sorted points: one CTA per brick stages the brick's
 * vertex tile in shared memory. brick_offsets from tgcu_sort_points, or NULL
 * (then computed by one extra pass over the points). Device pointers. */
int tgcu_eval_sorted(tgcu_grid* g, const float* sorted_pts, int64_t n, const int64_t* brick_offsets,
                     float* values, float* spatial_grad, int flags, void* stream);

/* backprop_value_and_spatial (taylor_grid.cpp:223-229), batched: adds
 * upstream[i]·∂f/∂c + upstream_vec[i]·∂∇f/∂c into grad (device, coeff_total
 * floats). upstream or upstream_vec may be NULL (= zeros; backprop_point /
 * backprop_spatial_chain, :205-221). */
int tgcu_backprop(tgcu_grid* g, const float* pts, const float* upstream, const float* upstream_vec,
                  int64_t n, float* grad, int flags, void* stream);

/* Device gradient buffer owned by the grid (coeff_total floats, zeroed at
 * creation). */
float* tgcu_grid_grad(tgcu_grid* g);
int tgcu_grad_zero(tgcu_grid* g, float* grad, void* stream); /* grad NULL: the grid's own buffer */
/* Copy a device gradient buffer (NULL = the grid's own) to host fp64. */
int tgcu_grad_download_f64(tgcu_grid* g, const float* grad, double* out, int64_t n);

/* tv_loss (sdf_loss.cpp:155-257). grad may be NULL (value only). */
/* recon_loss (sdf_loss.cpp:130-135): mean weighted L1 residual of the batch;
 * with grad (device, coefficient layout) the gradient times `scale` is added
 * into it. eikonal_loss (sdf_loss.cpp:137-153): mean (|grad f| - 1)^2 over
 * n points (n x 3 floats), gradient times `scale` added into grad. */
int tgcu_recon_loss(tgcu_grid* g, const float* samples, int64_t n, const tgcu_loss_config* cfg, double scale,
                    float* grad, double* out, int flags, void* stream);
int tgcu_eikonal_loss(tgcu_grid* g, const float* points, int64_t n, double scale, float* grad, double* out,
                      int flags, void* stream);
int tgcu_tv_loss(tgcu_grid* g, float* grad, double scale, double* out, void* stream);

/* total_loss (sdf_loss.cpp:259-292), reuse-batch eikonal: samples n×4
 * (x, y, z, gt). grad (device) may be NULL. Unfused path (gather, atomic
 * scatter into grad, then TV). */
int tgcu_total_loss(tgcu_grid* g, const float* samples, int64_t n, const tgcu_loss_config* cfg,
                    float* grad, tgcu_loss_terms* out, int flags, void* stream);

/* AdamState (adam.hpp:17-32): reset moments and t (AdamState::reset). */
int tgcu_adam_reset(tgcu_grid* g, const tgcu_adam_config* cfg);
int tgcu_adam_get_t(const tgcu_grid* g, int64_t* t);
/* adam_step (adam.cpp:12-56) on the grid's coefficients with grad (device):
 * non-finite grad -> TGCU_ERR_NUMERICAL naming the first index, params untouched. */
int tgcu_adam_step(tgcu_grid* g, const float* grad, void* stream);
/* Moment interop (reference layout, fp64 <-> fp32). */
int tgcu_adam_download_f64(tgcu_grid* g, double* m, double* v, int64_t n);

/* One fused training step = the run_schedule / cmd_bench inner loop
 * (schedule.cpp:66-92, tools/main.cpp:640-644): zero grad → total_loss →
 * finite-loss check → adam_step, as one device pipeline (point binning →
 * fused brick kernel → finalize). The gradient never touches HBM. On a
 * non-finite loss or gradient the step is not committed (params, moments and
 * t stay as before) and TGCU_ERR_NUMERICAL is returned (sticky under
 * TGCU_ASYNC; "stage 0 step k" / "index i" in the message). out may be NULL.
 * TGCU_HOST | TGCU_ASYNC with out == NULL pipelines host input: the samples are
 * copied on an internal copy stream into one of two device slots while the
 * previous step computes, and the step's LossTerms are copied back to pinned
 * host memory; the host array must stay valid and unmodified until
 * tgcu_sync() (its copy may still be in flight: do not refill one buffer for
 * consecutive steps).
 * Point binning runs on an internal stream into one of two bin sets, so the
 * binning of step i+1 overlaps step i's brick kernel when its input is known
 * complete (pipelined host input, or TGCU_INPUT_READY); otherwise it is
 * ordered after all earlier work on `stream`. */
int tgcu_train_step(tgcu_grid* g, const float* samples, int64_t n, const tgcu_loss_config* cfg,
                    tgcu_loss_terms* out, int flags, void* stream);
/* tgcu_train_step with EikonalPointSource::FreshUniform (sdf_loss.cpp:274-283):
 * the reconstruction term on the batch, the eikonal term on eik_points (n x 3
 * floats: the n points the reference draws per step with
 * rng->uniform_in_box(origin, domain_max), tgcu_rng_uniform_box), each
 * normalised by n; TV and Adam as tgcu_train_step. Host or device arrays per
 * TGCU_HOST; not pipelined. lambda1 == 0 draws nothing (plain train step). */
int tgcu_train_step_fresh_eik(tgcu_grid* g, const float* samples, int64_t n, const float* eik_points,
                              const tgcu_loss_config* cfg, tgcu_loss_terms* out, int flags, void* stream);
/* ---- multi-GPU z-slab training (owner computes) ----
 * A slab grid holds the brick layers [zb_lo, zb_hi) (bricks of 8^3 vertices)
 * of the global 3D spec: it owns (and Adam-updates) vertex planes
 * [8*zb_lo, min(8*zb_hi, res_z)) and stores one extra halo plane below and
 * above. A rank reads either the full global batch or only the points whose
 * cells touch its owned vertices (those in a slab-boundary cell layer belong
 * to both ranks); its binning keeps exactly those. A step is
 *   tgcu_slab_step_begin -> sum the 5 doubles at *partials over ranks
 *   (recon, eik, tv, nan flag, bad-grad flag; e.g. NCCL all-reduce in place)
 *   -> tgcu_slab_step_finish(reduced) -> exchange halo planes.
 * Gradients are never exchanged: each is computed by its owner; after the
 * commit each rank sends its boundary owned planes of the new parameters to
 * its neighbours (tgcu_slab_halo). Slab grids are training-only. */
int tgcu_grid_create_slab(const tgcu_grid_spec* global_spec, int zb_lo, int zb_hi, const tgcu_init_options* opts,
                          int device, tgcu_grid** out);
int tgcu_slab_info(const tgcu_grid* g, int* z_store_lo, int* z_store_n, int* z_own_lo, int* z_own_hi,
                   int* brick_layers);
/* samples: the n points this rank reads (the full global batch, or only the
 * points whose cells touch this slab's owned planes — slab.py
 * slab_point_mask); n_global: the global batch size for the loss scale 1/N
 * (<= 0: n). n may be 0 when n_global > 0 (a slab holding none of the
 * batch's points still applies TV and Adam to its vertices). */
int tgcu_slab_step_begin(tgcu_grid* g, const float* samples, int64_t n, int64_t n_global,
                         const tgcu_loss_config* cfg, double** partials, int flags, void* stream);
int tgcu_slab_step_finish(tgcu_grid* g, const double* reduced, tgcu_loss_terms* out, int flags, void* stream);
/* Device pointers (current parameters) of the planes to send to / receive
 * from the lower and upper neighbour (NULL at the grid boundary), and the
 * plane size in floats. */
int tgcu_slab_halo(tgcu_grid* g, float** send_lo, float** send_hi, float** recv_lo, float** recv_hi,
                   int64_t* plane_floats);

/* Fused halo (peer stores over NVLink): the brick kernel of the slab's lowest
 * and highest owned planes also writes those planes' new parameters straight
 * into the lower / upper neighbour's halo plane of the same ping-pong slot,
 * so no halo exchange follows the step. The per-step reduction of the partials
 * orders the neighbours (a rank's next step starts after every rank's brick
 * kernel has finished), and a rolled-back step leaves both sides' committed
 * slots untouched. Setup, once per run (slab.py SlabTrainer):
 *   tgcu_slab_ipc_export on every rank -> exchange the 144-byte blobs ->
 *   tgcu_slab_ipc_import(side 0, lower neighbour's blob),
 *   tgcu_slab_ipc_import(side 1, upper neighbour's blob) ->
 *   tgcu_slab_peer_probe(0) on every rank, barrier, tgcu_slab_peer_probe(1)
 *   (verifies the neighbours' writes landed); any failure -> keep exchanging.
 * blob: cudaIpcMemHandle_t of p[0] and p[1] (2 x 64 bytes), then the byte
 * offsets of this slab's lower and upper halo plane within them (2 x int64). */
int tgcu_slab_ipc_export(tgcu_grid* g, void* blob144);
int tgcu_slab_ipc_import(tgcu_grid* g, int side, const void* blob144);
/* Same-process form (one device hosting several slabs, tests): dst_lo[i] /
 * dst_hi[i] = the neighbour's halo plane in its slot-i parameters (NULL: no
 * neighbour on that side). */
int tgcu_slab_set_peer_planes(tgcu_grid* g, float* const dst_lo[2], float* const dst_hi[2]);
/* This slab's own halo planes (lower, upper; NULL at the grid boundary) in
 * parameter slots 0 and 1 — what a same-process neighbour passes above. */
int tgcu_slab_halo_slots(tgcu_grid* g, float* recv_lo[2], float* recv_hi[2]);
/* phase 0: write a probe pattern into the neighbours' halo planes of the
 * inactive slot; phase 1: check the neighbours' patterns in this slab's halo
 * planes (*ok = 1 when both sides match). Synchronous. */
int tgcu_slab_peer_probe(tgcu_grid* g, int phase, int* ok);

/* ---- communicator of a multi-GPU job (comm.cu; no PyTorch / MPI) ----------
 * One process per GPU. Rank 0 listens on addr:port and every other rank
 * connects (a TCP star that carries the bootstrap and the host-side
 * collectives). backend TGCU_COMM_NCCL: the slab step's all-reduce and halo
 * send/recv run as NCCL collectives on the step's stream (libnccl.so.2 is
 * loaded at run time); TGCU_COMM_HOST: the same collectives staged through
 * host memory over the star (tests, ranks sharing a device). Host
 * reductions combine the ranks in rank order (identical bits everywhere). */
enum { TGCU_COMM_NCCL = 0, TGCU_COMM_HOST = 1 };
typedef struct tgcu_comm tgcu_comm;
int tgcu_comm_create(const char* addr, int port, int rank, int nranks, int device, int backend, tgcu_comm** out);
int tgcu_comm_destroy(tgcu_comm* c);
int tgcu_comm_info(const tgcu_comm* c, int* rank, int* nranks, int* backend);
int tgcu_comm_barrier(tgcu_comm* c);
/* In-place reduction of n host doubles over the ranks: op 0 sum, 1 max, 2 min. */
int tgcu_comm_allreduce_host(tgcu_comm* c, double* buf, int n, int op);
/* out (nranks x bytes, rank order) receives every rank's `bytes` bytes. */
int tgcu_comm_allgather_host(tgcu_comm* c, const void* in, int64_t bytes, void* out);

/* Routed host point-to-point (collective: every rank calls it): send nsend
 * buffers to ranks dst[i]; receive nrecv buffers from ranks src[j] (sizes
 * must match; several messages from one rank arrive in send order). */
int tgcu_comm_exchange_host(tgcu_comm* c, int nsend, const int* dst, const void* const* sbuf, const int64_t* sbytes,
                            int nrecv, const int* src, void* const* rbuf, const int64_t* rbytes);

/* Attach a slab grid to the job: checks that the ranks' slabs tile the grid
 * in rank order, exchanges the initial halo planes, and (fused_halo != 0)
 * sets up the peer-memory halo (IPC handles over the star + probe round trip,
 * all ranks or none). *fused_out = 1 when the fused halo is active. */
int tgcu_slab_connect(tgcu_grid* g, tgcu_comm* c, int fused_halo, int* fused_out);
/* One slab training step over the attached communicator:
 * tgcu_slab_step_begin -> all-reduce of the 5 partials -> tgcu_slab_step_finish
 * -> halo planes (unless fused). Same flags / out semantics as
 * tgcu_train_step (TGCU_ASYNC with out == NULL: stream-ordered, no host sync
 * on the NCCL backend). */
int tgcu_slab_train_step(tgcu_grid* g, const float* samples, int64_t n, int64_t n_global,
                         const tgcu_loss_config* cfg, tgcu_loss_terms* out, int flags, void* stream);

/* ---- run_schedule on the device (schedule.hpp:13-86, schedule.cpp:13-108) ----
 * tg::Schedule::Stage, tg::TraceRow. */
typedef struct {
    int res[3];  /* vertices per axis (unused axes 2, as Stage's default) */
    int steps;
} tgcu_stage;
typedef struct {
    int64_t step;  /* global step index */
    int stage;
    int res[3];
    tgcu_loss_terms loss;
    double wall_ms;
} tgcu_trace_row;
/* The problem (tg::TrainProblem, schedule.hpp:60-66): the batch of a global
 * step — n x 4 floats (x, y, z, gt) in *samples, *flags = TGCU_HOST for host
 * memory (it may be refilled once the callback is called again), otherwise
 * device memory on the grid's device, written on `stream` (add
 * TGCU_INPUT_READY when it is already complete, so its binning can overlap
 * the previous step). Returns TGCU_OK or a status that aborts the run. */
typedef int (*tgcu_batch_fn)(void* user, tgcu_grid* g, int64_t global_step, const float** samples, int64_t* n,
                             int* flags);
/* TrainProblem::on_stage_start: after any upsample, before the stage's first step. */
typedef int (*tgcu_stage_fn)(void* user, tgcu_grid* g, int stage);
/* Schedule::validate (schedule.cpp:13-25), same messages. */
int tgcu_schedule_validate(const tgcu_stage* stages, int nstages, int dim);
/* Schedule::progressive (schedule.cpp:27-54): up to 3 stages into out. */
int tgcu_schedule_progressive(const int target[3], int dim, int total_steps, tgcu_stage out[3], int* nstages);
/* run_schedule (schedule.cpp:62-108): *grid is the stage-0 grid; on return it
 * is the final grid (upsampling replaces it: the previous handle is
 * destroyed). Each step is one fused device step (tgcu_train_step, reuse-batch
 * eikonal). flags TGCU_ASYNC: a stage's steps are issued without a host round
 * trip per step (windows of up to 4096, one sync each; wall_ms = the window's
 * mean). trace (total steps rows) and stage_seconds (nstages) may be NULL.
 * A non-finite loss -> TGCU_ERR_NUMERICAL "run_schedule: non-finite loss at
 * stage s step k", the grid at its last committed step. */
int tgcu_run_schedule(tgcu_grid** grid, const tgcu_stage* stages, int nstages, const tgcu_adam_config* adam,
                      const tgcu_loss_config* cfg, tgcu_batch_fn batch, tgcu_stage_fn on_stage, void* user, int flags,
                      void* stream, tgcu_trace_row* trace, double* stage_seconds);

/* Deterministic mode (the reference's --deterministic, run_config.cpp:239-242):
 * the fused step sums every gradient and loss partial in a canonical order
 * (each brick's binned points sorted by their bits, every cell run of a chunk
 * in record order), so repeated runs give bit-identical parameters and loss
 * traces. Costs a per-brick sort and per-cell run sorts per step; a brick may
 * then hold at most 4096 point copies (TGCU_ERR_CONFIG beyond). Default: off,
 * or on when the environment has TGCU_DETERMINISTIC=1 at grid creation. */
int tgcu_grid_set_deterministic(tgcu_grid* g, int on);

/* Fused-step path (no reference counterpart: an implementation choice behind
 * tgcu_train_step). TGCU_STEP_BRICK: binning + the brick kernel + finalize
 * (any grid). TGCU_STEP_SINGLE: the small-grid step, two launches chained
 * by programmatic dependent launch (thread per point with the gradients
 * reduced in L2, then thread per coefficient for TV + Adam + the commit) — for small grids such as BASELINE configs[0] (2D 128^2), where the
 * brick path's five launches are latency-bound. TGCU_STEP_AUTO (default)
 * takes it for grids of at most 3 x 2^20 coefficients and batches of at most
 * 2^22 points, and never for slab grids or in deterministic mode. Environment TGCU_STEP_PATH=brick|single at grid
 * creation sets the same. Results agree within the fused step's tolerances
 * (summation order of the gradient differs). */
#define TGCU_STEP_AUTO 0
#define TGCU_STEP_BRICK 1
#define TGCU_STEP_SINGLE 2
int tgcu_grid_set_step_path(tgcu_grid* g, int path);

/* CUDA-graph replay of small-grid training steps (no reference counterpart:
 * the reference's run_schedule loop, schedule.cpp:66-92, issued without a
 * host call per step). tgcu_train_graph_create captures nsteps (even, >= 2)
 * fused steps of the small-grid path on device batches samples[0..nsteps-1]
 * (n x 4 floats each, device pointers kept by the graph: refill their
 * contents between replays, ordered on the replay stream) on a non-default
 * stream; nothing runs at capture. tgcu_train_graph_launch replays them: the
 * same steps as nsteps tgcu_train_step(TGCU_ASYNC | TGCU_INPUT_READY) calls
 * (Adam t, trace rows and ping-pong slot advance on the device; errors are
 * sticky and reported by tgcu_sync, as for asynchronous steps). Fails with
 * TGCU_ERR_INVALID_ARGUMENT for a grid on the brick path (slab, deterministic,
 * large grids or TGCU_STEP_BRICK), an odd nsteps, or a replay after an odd
 * number of other steps. */
typedef struct tgcu_graph tgcu_graph;
int tgcu_train_graph_create(tgcu_grid* g, const float* const* samples, int nsteps, int64_t n,
                            const tgcu_loss_config* cfg, void* stream, tgcu_graph** out);
int tgcu_train_graph_launch(tgcu_graph* graph, void* stream);
int tgcu_train_graph_destroy(tgcu_graph* graph);

/* Collective phase of the profiled slab steps (those whose brick kernel
 * tgcu_profile_begin / _every times): summed device ms of the all-reduce of
 * the partials and of the halo exchange (0 with the fused peer-memory halo,
 * whose stores run inside the brick kernel), and the number of steps. Resets. */
int tgcu_slab_comm_profile(tgcu_grid* g, double* allreduce_ms, double* halo_ms, int* steps);

/* Fused steps issued on this grid since creation or the last reported error;
 * error messages of a failed step name it as "step <this index at launch>". */
int tgcu_grid_steps_launched(const tgcu_grid* g, int64_t* n);

/* Wait for the grid's outstanding async work and report any sticky error.
 * If last_terms is not NULL it receives the most recent step's LossTerms. */
int tgcu_sync(tgcu_grid* g, tgcu_loss_terms* last_terms);
/* Per-step LossTerms of the last `count` async steps (oldest first, up to the
 * trace capacity of 4096). */
int tgcu_trace(tgcu_grid* g, tgcu_loss_terms* out, int count);

/* Live timing of the fused brick kernel: CUDA events recorded on the launch
 * stream around every k_brick_step launch between begin and end; end returns
 * the summed device milliseconds and the number of timed launches. */
/* Diagnostics: enable = 1 starts recording events at the boundaries of each
 * fused step (synchronising after each step); enable = 0 stops and returns the
 * mean ms of {brick histogram, column pass, scatter, brick kernel, finalize}. */
int tgcu_step_breakdown(tgcu_grid* g, int enable, double* mean_ms5, int* steps);
int tgcu_profile_begin(tgcu_grid* g);
/* Time only every `every`-th fused brick launch (events around a launch cost
 * the stream ~3 us each); tgcu_profile_end then reports the sampled launches. */
int tgcu_profile_every(tgcu_grid* g, int every);
int tgcu_profile_end(tgcu_grid* g, double* total_ms, int* launches);

/* ---- stage transitions, lattice query, .tgrid I/O ---------- */

/* multilinear_resample (taylor_grid.cpp:231-271): `channels` interleaved values
 * per vertex of old_spec (n = vertex_count * channels floats) resampled onto
 * new_res (per-axis vertex counts of the same origin/extent). Weights and
 * accumulation in fp64 in the reference's order, rounded once to fp32. data /
 * out are device pointers, or host with TGCU_HOST. */
int tgcu_multilinear_resample(const tgcu_grid_spec* old_spec, const float* data, int64_t n, int channels,
                              const int new_res[3], float* out, int flags, void* stream);

/* upsample (taylor_grid.cpp:273-284) into an existing grid: dst must have
 * src's dim, order, origin and extent, and res >= src's on every axis
 * (TGCU_ERR_INVALID_ARGUMENT "upsample: resolution may not shrink (axis a)").
 * dst's coefficients are replaced; its Adam state is the caller's to reset
 * (run_schedule resets moments per stage, schedule.cpp:79). */
int tgcu_grid_upsample(tgcu_grid* src, tgcu_grid* dst, int flags, void* stream);

/* sample_grid_field (marching.cpp:53-58): eval on the lattice[0] x lattice[1]
 * (x lattice[2] in 3D) points origin + extent * i / (lattice - 1) of the
 * grid's own domain (ScalarField3::position, marching.hpp:21-24), x fastest.
 * For dim 2 this is the CLI's sample_grid_field2 (tools/main.cpp:33-45).
 * values: device (or host with TGCU_HOST) array of prod(lattice) floats. */
int tgcu_sample_grid_field(tgcu_grid* g, const int lattice[3], float* values, int flags, void* stream);

/* tg::IouOptions (metrics.hpp:12-18). */
typedef struct {
    int64_t samples;  /* default 100000 */
    uint64_t seed;    /* default 7 */
    double lo[3];     /* default (-1, -1, -1) */
    double hi[3];     /* default (1, 1, 1) */
    int dim;          /* default 3 */
} tgcu_iou_options;
/* iou (metrics.cpp:104-124): Monte-Carlo IoU of {a < 0} and {b < 0} on the
 * reference's point stream (Rng(seed).uniform_in_box, drawn in order); a is
 * evaluated on the device; b is grid b or, when b is NULL, the sphere
 * |p| - sphere_radius (cmd_bench's probe target). *empty_union = 1 (iou 1)
 * when neither set has a sample. */
int tgcu_iou(tgcu_grid* a, tgcu_grid* b, double sphere_radius, const tgcu_iou_options* o, double* iou,
             int* empty_union);

/* SdfProblem::compute's batch draw (sdf_fit.cpp:21-23) on device: n samples
 * (x, y, z, gt) drawn with replacement from a device pool of pool_n samples,
 * index = floor(u * pool_n), u from a counter hash of (seed, step, i) — a
 * different stream from the reference's mt19937_64, same distribution. */
int tgcu_draw_batch(const float* pool, int64_t pool_n, int64_t n, uint64_t seed, uint64_t step, float* out,
                    void* stream);

/* tg::Rng streams (rng.hpp:14-74, mt19937_64 + the reference's index()
 * rejection mapping) as host handles, for drivers that need the reference's
 * exact draw sequence: SdfProblem's batch indices (sdf_fit.cpp:22). */
typedef struct tgcu_rng tgcu_rng;
int tgcu_rng_create(uint64_t seed, tgcu_rng** out);
void tgcu_rng_destroy(tgcu_rng* r);
/* count draws of Rng::index(n) into out. */
int tgcu_rng_index(tgcu_rng* r, uint64_t n, int64_t count, int64_t* out);
/* Rng::uniform_in_box (rng.hpp:53-57): count points, axes 0..dim-1 drawn in
 * order from [lo, hi), z = 0 in 2D, into out3 (count x 3 doubles). */
int tgcu_rng_uniform_box(tgcu_rng* r, int dim, const double* lo, const double* hi, int64_t count, double* out3);
/* fit_sdf's seeded Fisher-Yates order (sdf_fit.cpp:59-64); pass the
 * reference's seed (options.seed ^ 0x5deece66d). */
int tgcu_shuffle_order(uint64_t seed, int64_t n, uint32_t* order);

/* ---- radiance density chain (volume_render.cpp:61-276, sh.cpp:43-107) ---- */
enum { TGCU_DENSITY_SHIFTED_SOFTPLUS = 0, TGCU_DENSITY_CLAMP_RELU = 1 };
/* tg::RenderOptions (volume_render.hpp:17-24). */
typedef struct {
    int n_samples;          /* 1..1024 samples per ray, t_i = near + i (far - near) / n */
    int activation;         /* TGCU_DENSITY_* (apply_activation, volume_render.cpp:19-28) */
    double softplus_shift;  /* default -10 */
    double background[3];   /* default (1, 1, 1) */
    int jitter;             /* stratified jitter: t_i = near + (i + u_i) (far - near) / n with u_i the
                               ray's own Rng stream (volume_render.cpp:69-70), ray id = batch index */
    uint64_t jitter_seed;
} tgcu_render_options;
/* photometric_loss (volume_render.cpp:210-276) / render_ray (:194-208),
 * batched: the density is `density` (3D TaylorGrid, current parameters); the
 * color an SH grid (tg::SHColorGrid, sh.hpp:19-29) of geometry sh_spec, degree
 * 0..2, coefficients sh_coeffs (vertex-major, [R basis | G basis | B basis]).
 * rays: n x 8 floats (origin xyz, unit direction xyz, near, far), 16-byte
 * aligned; gt: n x 3 or NULL (render only). Outputs (each may be NULL): colors
 * n x 3, residual transmittance n, loss = mean squared RGB error; gradients
 * accumulate (+=) into grad_density (coeff_total) and grad_sh (SH coeffs).
 * Device pointers, or host with TGCU_HOST. A NaN ray -> INVALID_ARGUMENT. */
int tgcu_photometric_loss(tgcu_grid* density, const tgcu_grid_spec* sh_spec, int sh_degree, const float* sh_coeffs,
                          const float* rays, const float* gt, int64_t n, const tgcu_render_options* opts,
                          float* colors, float* residual, float* grad_density, float* grad_sh, double* loss,
                          int flags, void* stream);

/* .tgrid files (grid_io.cpp:36-111, layout grid_io.hpp:11-16). F64 writes the
 * fp32 coefficients widened (exact); loading an F64 file narrows to fp32.
 * File errors -> TGCU_ERR_INGEST with the reference's messages. */
enum { TGCU_TGRID_F64 = 0, TGCU_TGRID_F32 = 1 };
int tgcu_save_tgrid(tgcu_grid* g, const char* path, int precision);
int tgcu_load_tgrid(const char* path, int device, tgcu_grid** out);
/* tgrid_file_size (grid_io.cpp:36-40); -1 for an invalid spec. */
int64_t tgcu_tgrid_file_size(const tgcu_grid_spec* spec, int precision);

/* Pinned (page-locked) host memory for batches fed through the pipelined
 * host path (TGCU_HOST | TGCU_ASYNC); pageable memory is copied synchronously. */
int tgcu_host_alloc(void** p, size_t bytes);
int tgcu_host_free(void* p);

/* Number of kernels this library launched since the counter was reset. */
int64_t tgcu_launch_count(void);
void tgcu_reset_launch_count(void);

/* Host-side seeded input generation with the reference Rng semantics
 * (rng.hpp:14-74): mt19937_64, uniform = (x>>11)·2^-53, Box–Muller gaussian.
 * shape: 0 = sphere r=param0 (3D), 1 = 2D circle r=0.5 ∪ box (BASELINE C1),
 * 2 = procedural min-union of 64 seeded primitives (C3/C5).
 * Writes n×4 floats (x, y, z, gt). near_frac of the points are near-surface
 * (surface point + N(0, sigma) per axis, clamped), the rest uniform in the
 * domain box (uniform first, as sample_sphere_points, sampling.cpp:94-103). */
int tgcu_sample(int shape, int dim, uint64_t seed, int64_t n, double near_frac, double sigma,
                double param0, float* out4);
/* Device-side uniform points in [lo, hi]^dim from a counter hash (n×3,
 * device pointer; z = 0 in 2D). For large synthetic query sets. */
int tgcu_sample_uniform_device(int dim, uint64_t seed, int64_t n, double lo, double hi, float* out3,
                               void* stream);
/* Uniform query points in [lo, hi]^dim (n×3, z = 0 in 2D). */
int tgcu_sample_uniform(int dim, uint64_t seed, int64_t n, double lo, double hi, float* out3);
/* Analytic target SDF of a shape at points (n×3 fp64 in, n out). */
int tgcu_shape_sdf(int shape, int dim, double param0, const double* pts, int64_t n, double* out);

#ifdef __cplusplus
}
#endif

#endif /* TGCU_H */
