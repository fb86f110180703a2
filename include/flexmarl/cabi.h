/* include/flexmarl/cabi.h — the C ABI of the B200 micro-batch policy-update path.
 *
 * The reference (FlexMARL artifact, /root/reference/proj/include/marlsim) has
 * no FFI: its hot path sits behind C++ class methods in header-only code.
 * This ABI is what those methods bind to in the drop-in replacement
 * (INTEGRATION.md shows the reference-side C++ shim and the ctypes binding).
 * Each entry point names the reference interface it replaces (file:line,
 * paths relative to proj/include/marlsim/).
 *
 * Conventions: plain pointers and sizes, no exceptions across the boundary;
 * every call returns an fm_status (0 = OK) and sets a thread-local message
 * readable with fm_last_error().  Status codes 1..28 are marlsim::ErrorCode
 * (errors.hpp:10-39) + 1, so the C++ shim can re-raise them verbatim.
 * Calls on one fm_ctx come from one host thread (the reference is a
 * single-threaded event loop by contract, sim.hpp:19-23).
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point fails with FM_ERR_NO_DEVICE.
 */
#ifndef FLEXMARL_CABI_H
#define FLEXMARL_CABI_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fm_status {
    FM_OK = 0,
    /* marlsim::ErrorCode + 1 (errors.hpp:10-39) */
    FM_ERR_SCHEDULING_IN_PAST = 1,
    FM_ERR_DEVICE_OOM = 2,
    FM_ERR_HOST_OOM = 3,
    FM_ERR_EMPTY_POOL = 4,
    FM_ERR_DUPLICATE_KEY = 5,
    FM_ERR_KEY_NOT_FOUND = 6,
    FM_ERR_GET_TIMEOUT = 7,
    FM_ERR_LAYOUT_OUT_OF_BOUNDS = 8,
    FM_ERR_EMPTY_LIST = 9,
    FM_ERR_TABLE_EXISTS = 10,
    FM_ERR_RESERVED_COLUMN_NAME = 11,
    FM_ERR_DUPLICATE_SAMPLE = 12,
    FM_ERR_UNKNOWN_COLUMN = 13,
    FM_ERR_RECORD_NOT_FOUND = 14,
    FM_ERR_CELL_ALREADY_SET = 15,
    FM_ERR_UNKNOWN_TABLE = 16,
    FM_ERR_NOT_PROCESSING = 17,
    FM_ERR_BAD_SAMPLE_ID = 18,
    FM_ERR_UNKNOWN_WORKFLOW = 19,
    FM_ERR_NO_INSTANCE = 20,
    FM_ERR_INSUFFICIENT_RESOURCES = 21,
    FM_ERR_BUSY_GROUP = 22,
    FM_ERR_VERSION_MISMATCH = 23,
    FM_ERR_INACTIVE_GROUP = 24,
    FM_ERR_INCOMPLETE_BATCH = 25,
    FM_ERR_CONFIG_ERROR = 26,
    FM_ERR_STALL_DETECTED = 27,
    FM_ERR_SYNC_TIMEOUT = 28,
    /* B200 runtime */
    FM_ERR_CUDA = 100,
    FM_ERR_NCCL = 101,
    FM_ERR_NO_DEVICE = 102,
    FM_ERR_INVALID_ARG = 103
} fm_status;

/* Arithmetic of an agent's trainer (declared per agent). */
typedef enum fm_precision {
    FM_PRECISION_BF16_TC = 0,  /* tcgen05 bf16 GEMMs, fp32 accumulate, fp64 master weights */
    FM_PRECISION_PARITY_F64 = 1 /* exact-featurizer fp64 SIMT path (correctness anchor, small V*D) */
} fm_precision;

/* Where a suspended agent's training state is parked (object_store.hpp:80-86 tiers). */
typedef enum fm_tier {
    FM_TIER_HOST = 0,   /* pinned host memory of this process (D2H / H2D copies) */
    FM_TIER_DEVICE = 1, /* a parking arena in this GPU's HBM (D2D copy engine) */
    FM_TIER_PEER = 2    /* a peer GPU's HBM over NVLink (cudaMemcpyPeerAsync) */
} fm_tier;

typedef struct fm_ctx fm_ctx;     /* one GPU: streams, token arena, workspace */
typedef struct fm_agent fm_agent; /* one agent's trainer state (training.hpp:98-105) */
typedef struct fm_store fm_store; /* host control plane of the experience store */
typedef struct fm_comm fm_comm;   /* NCCL communicator of one agent gang */

/* ---- misc ------------------------------------------------------------- */
const char* fm_last_error(void);
const char* fm_status_name(int status);
int fm_abi_version(void);
/* Number of hot-path kernel launches issued by this process so far. */
uint64_t fm_launch_count(void);

/* ---- host-side bit-exact helpers (rng.hpp, policy.hpp, training.hpp) --- */
/* training.hpp:245-248: mix_str(mix_u64(seed, 0x1217), agent) */
uint64_t fm_agent_seed(uint64_t seed, const char* agent);
/* policy.hpp:29-35 PolicyModel::seeded, bit-identical (host glibc libm), multi-threaded */
int fm_seeded_weights(uint64_t V, uint64_t D, uint64_t seed, double* out, int threads);
/* codec.hpp:15-22 encode_tokens; returns bytes written (8 + 8n) */
uint64_t fm_encode_tokens(const int32_t* tokens, uint64_t n, uint8_t* out);

/* ---- device context ------------------------------------------------------ */
int fm_ctx_create(int device, fm_ctx** out);
int fm_ctx_destroy(fm_ctx* ctx);
int fm_ctx_device(const fm_ctx* ctx);
int fm_ctx_num_sms(const fm_ctx* ctx);
int fm_ctx_synchronize(fm_ctx* ctx);
/* Device step timer on the compute stream (copy streams joined at stop). */
int fm_ctx_timer_start(fm_ctx* ctx);
int fm_ctx_timer_stop(fm_ctx* ctx, double* ms);
/* Per-kernel CUDA-event timing of the hot path (off by default).  Kinds (8 slots):
 * 0 gather (K-gather + K-pos + K-pslot), 1 stats (K-stats), 2 lse, 3 band (K-band),
 * 4 gemm2, 5 adam, 6 parity, 7 memset. */
int fm_ctx_set_kernel_timing(fm_ctx* ctx, int on);
int fm_ctx_kernel_times(fm_ctx* ctx, double* ms_out, int64_t* count_out, int reset);
/* Pre-size the token arena and the per-micro-batch workspace. */
int fm_ctx_reserve(fm_ctx* ctx, uint64_t arena_bytes, int64_t max_rows, uint64_t max_vocab,
                   uint64_t max_feat);

/* ---- token arena: the device side of ObjectStore::set/get for the List
 * cells "prompt"/"response" (object_store.hpp:116-197, codec.hpp:15-30).
 * fm_arena_put uploads one encoded token list and returns its arena offset. */
int fm_arena_put(fm_ctx* ctx, const uint8_t* payload, uint64_t nbytes, uint64_t* offset_out);
int fm_arena_reset(fm_ctx* ctx);
uint64_t fm_arena_used(const fm_ctx* ctx);

/* ---- agent trainer (TrainingEngine, training.hpp:192-540) ----------------- */
int fm_agent_create(fm_ctx* ctx, const char* agent, uint64_t vocab, uint64_t feat,
                    int precision, fm_agent** out);
int fm_agent_destroy(fm_agent* a);
/* initial_model / peek_state (training.hpp:224-248): V*D f64 row-major */
int fm_agent_set_weights(fm_agent* a, const double* W);
int fm_agent_read_weights(fm_agent* a, double* W_out);
/* Adam moments (fp32 on device) and step count (training.hpp:31-35) */
int fm_agent_read_moments(fm_agent* a, float* m_out, float* v_out, int64_t* step_out);
/* gradient accumulator (V*D, as f64) — the reduced -1/G * sum term of training.hpp:444-446 */
int fm_agent_read_grad(fm_agent* a, double* g_out);
/* the same, as the device holds it (fp32, tensor-core agents): V*D floats, half the host memory */
int fm_agent_read_grad_f32(fm_agent* a, float* g_out);
/* selected feature columns of the gradient accumulator, [V][n_cols] row-major as f64
 * (parity tooling at full V x D, where reading all V*D is host-memory heavy) */
int fm_agent_read_grad_cols(fm_agent* a, const int64_t* cols, int64_t n_cols, double* g_out);
/* K rows the segmented K-GEMM2 launches on ctx ran since the last reset, summed
 * over their 256-feature column blocks (executed flops = 2 * V * 256 * rows);
 * reset != 0 zeroes the counter after reading. */
int fm_ctx_gemm2_rows(fm_ctx* c, int64_t* rows_out, int reset);
/* kernel test hook (device pointers): C[M][N] fp32 = sum_k A(m,k) B(n,k) through the
 * tcgen05 CTA-pair GEMM, A/B K-major ([M][K] / [N][K]) or MN-major ([K][M] / [K][N]) */
int fm_debug_gemm(fm_ctx* c, const void* A, const void* B, int a_mn, int b_mn, int M, int N, int K, float* C);
int64_t fm_agent_version(const fm_agent* a);
int64_t fm_agent_samples_accumulated(const fm_agent* a);
int fm_agent_is_active(const fm_agent* a);

/* One polled record as handed to the trainer (sample.hpp:94-111): arena
 * offsets of its prompt / response payloads and its advantage cell. */
typedef struct fm_sample {
    uint64_t prompt_off;
    uint64_t response_off;
    double advantage;
} fm_sample;

/* Same, with host payload pointers (end-to-end path: the ABI stages the
 * encoded lists through pinned memory into the arena inside the call). */
typedef struct fm_host_sample {
    const uint8_t* prompt;
    const uint8_t* response;
    double advantage;
} fm_host_sample;

/* Completion record of one micro-batch (GradReport, training.hpp:169-177). */
typedef struct fm_report {
    int64_t ticket;
    int64_t tokens;
    int64_t batch_size;
    double grad_norm; /* ||sum_mb A_i term_i|| / G (training.hpp:417); NaN under DP unless fm_agent_set_dp_norms */
    double loss;      /* -(1/G) sum_i A_i sum_t log pi, this micro-batch */
} fm_report;

/* Identity of a trained sample: GradKey (training.hpp:87-91) = sample id
 * (input_id, number_of_turns, trajectory_id; sample.hpp:38-47) + the policy
 * version it was generated under. */
typedef struct fm_sample_key {
    const char* input_id;
    int32_t turns;
    int32_t traj;
    int64_t version;
} fm_sample_key;

/* DuplicateSample guard of train_micro_batch (training.hpp:396-401): adds the
 * micro-batch's keys to the agent's set for the current global step, or fails
 * with FM_ERR_DUPLICATE_SAMPLE (nothing added) if any key is already there or
 * repeats in the list.  apply_global_update clears the set (training.hpp:448).
 * Callers: before fm_train_micro_batch of the same samples. */
int fm_agent_add_grad_keys(fm_agent* a, const fm_sample_key* keys, int n);

/* TrainingEngine::train_micro_batch (training.hpp:355-430): gather -> positions ->
 * K-stats -> K-lse -> K-band enqueued on the agent's stream; the weight-gradient
 * GEMM is queued and runs once for the step's queued micro-batches (at the step's
 * last micro-batch, when 4 are queued, or when anything needs the agent's dW or a
 * queued report: fm_agent_sync, fm_agent_poll_report of that ticket, any other
 * call on the agent, another agent's micro-batch on the context).
 * Returns immediately; *ticket_out identifies the report (fm_agent_poll_report).
 * global_batch is G of the -1/G normalisation (training.hpp:446). */
int fm_train_micro_batch(fm_agent* a, const fm_sample* samples, int n, int64_t global_batch,
                         int64_t* ticket_out);
int fm_train_micro_batch_host(fm_agent* a, const fm_host_sample* samples, int n,
                              int64_t global_batch, int64_t* ticket_out);
/* Optional PPO clipped-ratio surrogate (off by default = the reference's
 * ratio-free objective).  old_logp: per packed row of the next
 * micro-batch (host array, n_rows entries = all its rows, also under DP) or NULL
 * to disable; the next train call fails with FM_ERR_INVALID_ARG if n_rows
 * differs from its row count. */
int fm_agent_set_clip(fm_agent* a, float clip_eps, const float* old_logp, int64_t n_rows);
/* Data-parallel gang: every rank receives the whole micro-batch and trains
 * the token-balanced row range [M*rank/nranks, M*(rank+1)/nranks). */
int fm_agent_set_shard(fm_agent* a, int rank, int nranks);
/* Per-row log pi(a_t|s_t) of the last micro-batch (f32; f64 in parity mode). */
int fm_agent_read_logp(fm_agent* a, double* out, int64_t n_rows);
/* Packed rows of the last micro-batch on ctx (the device gather's output,
 * bit-exact target of the oracle's fmo_pack_rows); any pointer may be NULL. */
int fm_debug_read_rows(fm_ctx* ctx, int64_t n_rows, int32_t* action, int32_t* ctx4,
                       int32_t* n_ctx, int32_t* sample, float* coef);
/* Context positions of the last tensor-core micro-batch on ctx (the band
 * formulation): each row's first position, each position's
 * feature (tok mod D, -1 before a sequence start) and K-GEMM2 segment slot. */
int fm_debug_read_positions(fm_ctx* ctx, int64_t n_rows, int32_t* q0, int64_t n_pos, int32_t* feat, int32_t* slot);
/* Runs the agent's queued gradient GEMM, then blocks until its stream drains;
 * every report becomes pollable. */
int fm_agent_sync(fm_agent* a);
/* Non-blocking: 1 and fills *out if the ticket's micro-batch has finished (a
 * queued gradient GEMM of that micro-batch is launched first). */
int fm_agent_poll_report(fm_agent* a, int64_t ticket, fm_report* out);

/* apply_global_update (training.hpp:435-456): IncompleteBatch unless
 * samples_accumulated == global_batch; fused Adam; version += 1.
 * If grad_norm_out != NULL the call waits and writes ||grad||_F. */
int fm_apply_update(fm_agent* a, int64_t global_batch, double lr, double beta1, double beta2,
                    double eps, double* grad_norm_out, int64_t* version_out);
/* apply_global_update followed by suspend(FM_TIER_DEVICE) (training.hpp:435-456,
 * 321-350), fused: K-adam writes the updated state straight into the agent's
 * parking buffer on its GPU, so no copy-out pass runs; fm_agent_activate
 * brings it back as after fm_agent_suspend.  Tensor-core agents outside a gang. */
int fm_apply_update_park(fm_agent* a, int64_t global_batch, double lr, double beta1, double beta2,
                         double eps, double* grad_norm_out, int64_t* version_out);

/* ---- training-state swap (suspend / activate, training.hpp:259-350) -------
 * suspend: copy {W, m, v, accumulated gradient} to the parking tier on the
 * ctx's copy stream (ordered after the agent's compute) and release the
 * agent's slot; activate: copy back into a slot of `ctx` (may differ from the
 * one it was suspended from), regenerate the bf16 shadow.  Both are async;
 * compute issued after activate waits on the copy-in event. */
int fm_agent_suspend(fm_agent* a, int tier, int peer_device);
int fm_agent_activate(fm_agent* a, fm_ctx* ctx);
/* FNV-1a over the bytes of {W, m, v, grad, step, version, samples}: swap-identity check. */
int fm_agent_state_checksum(fm_agent* a, uint64_t* out);

/* ---- migration between GPUs of different processes (SURVEY §8e agents <-> GPUs) ----
 * The location-agnostic swap (training.hpp:259-350) across the one-process-per-GPU
 * layout.  export lends the agent's live training slot: it writes a blob (CUDA IPC
 * handles of the slot and of an interprocess event recorded after the agent's
 * queued compute, plus version / Adam step / accumulated samples) and the agent
 * becomes inactive; the caller ships the blob to the target process (any side
 * channel), whose import pulls the state into an agent of the same shape that is
 * active on its GPU (e.g. fresh from fm_agent_create) with copy-engine NVLink peer
 * copies on its copy stream, blocking the host until they land.  After the import
 * returned, the sender calls migrate_release (or destroy) to return the slot. */
int fm_agent_migrate_export(fm_agent* a, uint8_t* blob_out, uint64_t cap, uint64_t* len);
int fm_agent_migrate_import(fm_agent* a, fm_ctx* ctx, const uint8_t* blob, uint64_t len);
/* Import only vocabulary rows [row_lo, row_hi) of W / m / v (and of a pending dW) plus the
 * whole shadow: for a rank joining a vocabulary-parallel gang, which keeps only its own rows
 * current (fm_gang_attach_mode 1 checks the range; until then, and unless a later
 * fm_gang_gather_state completes it, every other use of the agent fails ConfigError). */
int fm_agent_migrate_import_rows(fm_agent* a, fm_ctx* ctx, const uint8_t* blob, uint64_t len, uint64_t row_lo,
                                 uint64_t row_hi);
int fm_agent_migrate_release(fm_agent* a);
/* Same blob, the agent stays active here: several processes may import it (a DP
 * gang forming around the agent); no work may be queued for it until every
 * importer returned. */
int fm_agent_share_export(fm_agent* a, uint8_t* blob_out, uint64_t cap, uint64_t* len);

/* ---- weight publish / rollout sync ----------------------------
 * publish_weights (training.hpp:459-467): one contiguous device buffer in
 * pack_weights' single-tensor layout (object_store.hpp:258-273), stamped with
 * the agent version.  dtype 0 = f64 (reference payload bytes), 1 = f32, 2 = bf16,
 * 3 = f64 transposed [D][V] (rollout layout for fm_generate: coalesced feature reads). */
typedef struct fm_weights fm_weights;
int fm_publish_weights(fm_agent* a, int dtype, fm_weights** out);
/* Republish the agent's current weights into an existing buffer (same V x D,
 * dtype from the buffer): the allocation-free steady-state path. */
int fm_publish_into(fm_agent* a, fm_weights* w);
int fm_weights_alloc(fm_ctx* ctx, uint64_t rows, uint64_t cols, int dtype, fm_weights** out);
int fm_weights_info(const fm_weights* w, int64_t* version, uint64_t* rows, uint64_t* cols, int* dtype,
                    uint64_t* nbytes, int* device);
/* One Get per rollout consumer (rollout.hpp:510-541): host (dst_device -1) or any GPU (NVLink P2P);
 * synchronous (returns when the copy has landed), keeps the caller's current device. */
int fm_weights_get(const fm_weights* w, void* dst, int dst_device);
/* Sync every rank of a communicator from `root` in one NCCL broadcast (NVLink/NVSwitch). */
int fm_weights_broadcast(fm_weights* w, fm_comm* c, int root);
int fm_weights_destroy(fm_weights* w);

/* ---- rollout generation on the GPU ----------------------------
 * PolicyModel::generate (policy.hpp:119-130) for n requests from a published
 * f64 weight buffer (dtype 0 or 3) on ctx's GPU: request i has prompt
 * prompts[prompt_off[i]:prompt_off[i+1]] and token seed seeds[i] (the
 * reference derives it as rollout.hpp:640-644); outputs are n x max_tokens
 * row-major (tokens, log pi) and per-request lengths (EOS included). */
int fm_generate(fm_ctx* ctx, const fm_weights* w, const int32_t* prompts, const int32_t* prompt_off, int n,
                int max_tokens, const uint64_t* seeds, int32_t* out_tokens, double* out_logp,
                int32_t* out_len);

/* ---- PolicyState wire format (training.hpp:107-164) -----------
 * Byte-identical to PolicyState::serialize when no gradient is pending; a
 * pending step is one cache entry ("__sum__",0,0,version) holding sum(term).
 * out == NULL returns the required length.  deserialize reads matrix dims in
 * the defined rows-then-cols order (training.hpp:146 evaluates them in
 * unspecified order and transposes W when V != D). */
int fm_agent_serialize(fm_agent* a, int64_t global_batch, uint8_t* out, uint64_t cap, uint64_t* len);
int fm_agent_deserialize(fm_agent* a, int64_t global_batch, const uint8_t* in, uint64_t len);

/* ---- GRPO advantages (training.hpp:54-67), device kernel K-adv --------------
 * rewards[seg_off[i]:seg_off[i+1]] is group i; host arrays in/out. */
int fm_group_advantages(fm_ctx* ctx, const double* rewards, const int32_t* seg_off, int nseg,
                        double eps, double* out);

/* ---- data-parallel gang (NCCL over NVLink) ------------------------------- */
int fm_comm_unique_id(uint8_t out[128]);
int fm_comm_create(fm_ctx* ctx, const uint8_t id[128], int nranks, int rank, fm_comm** out);
int fm_comm_destroy(fm_comm* c);
/* Exact per-micro-batch grad norm under DP (training.hpp:417), opt-in
 * diagnostic: each micro-batch's contribution is all-reduced over `c` (the
 * gang's communicator) and measured, so fm_report.grad_norm is the reference's
 * value instead of NaN.  Costs a P-float all-reduce per micro-batch.  NULL
 * turns it off.  Collective: every rank of the gang calls it. */
int fm_agent_set_dp_norms(fm_agent* a, fm_comm* c);
/* Sum the agent's gradient accumulator across the gang (before fm_apply_update).
 * A no-op for agents attached with fm_gang_attach (reduced inside GEMM2). */
int fm_agent_allreduce_grad(fm_agent* a, fm_comm* c);
/* Fused GEMM2 -> reduce-scatter over NVLink peer memory + sharded Adam with
 * the bf16 all-gather fused into it.  attach writes this rank's
 * export blob (blob_out NULL -> just *len); the caller all-gathers the blobs
 * across the gang (any side channel) and passes them, in rank order, to
 * connect.  While attached the agent trains token-balanced row shards and its
 * master W / m / v rows outside its own shard are not maintained. */
int fm_gang_attach(fm_agent* a, fm_comm* c, uint8_t* blob_out, uint64_t cap, uint64_t* len);
/* Same with a mode: 0 = the token-sharded gang above; 1 = vocabulary-parallel:
 * every rank trains ALL rows of each micro-batch on its vocabulary range of
 * 256-row shards — K-stats / K-band on its columns, K-GEMM2 / K-adam on its rows
 * of dW / W, its own W16^T columns — so no partial gradients cross NVLink; per
 * micro-batch the rows' partial softmax sums and taken-token logits (2 floats per
 * row) and the squared gradient norm are all-reduced (the micro-batch grad norm
 * is the reference's, training.hpp:417).  The per-feature softmax bound is
 * max-all-reduced once per update.  Same blob / connect / detach protocol. */
int fm_gang_attach_mode(fm_agent* a, fm_comm* c, int mode, uint8_t* blob_out, uint64_t cap, uint64_t* len);
int fm_gang_connect(fm_agent* a, const uint8_t* blobs, uint64_t blob_len);
int fm_gang_detach(fm_agent* a);
/* Before a gang dissolves: pull the peers' W / m / v rows (the sharded Adam keeps
 * only the own rows current) into this rank's slot over NVLink, so that after
 * detach this rank holds the whole training state.  All gang ranks idle. */
int fm_gang_gather_state(fm_agent* a);

/* ---- experience store host control plane (experience_store.hpp:19-276) ---- */
int fm_store_create(fm_store** out);
int fm_store_destroy(fm_store* s);
/* column types: ColumnType (sample.hpp:69): 0 Int 1 Float 2 Bool 3 String 4 List 5 Tensor */
int fm_store_create_table(fm_store* s, const char* agent, const char* const* col_names,
                          const int* col_types, int ncols);
int fm_store_insert(fm_store* s, const char* agent, int64_t version, const char* input_id,
                    int turns, int traj);
int fm_store_set_float(fm_store* s, const char* agent, const char* input_id, int turns, int traj,
                       int64_t version, const char* column, double value);
/* set_cell_payload (experience_store.hpp:82-88): the payload goes to ctx's
 * token arena; the cell records its arena offset as the reference key. */
int fm_store_set_payload(fm_store* s, fm_ctx* ctx, const char* agent, const char* input_id,
                         int turns, int traj, int64_t version, const char* column,
                         const uint8_t* payload, uint64_t nbytes);
/* ready_count (experience_store.hpp:181-187) */
int fm_store_ready_count(fm_store* s, const char* agent, int64_t version, uint64_t* out);
int fm_store_record_count(fm_store* s, const char* agent, uint64_t* out);
/* poll_micro_batch (experience_store.hpp:92-114): canonical-first mb ready
 * records; writes mb samples (prompt/response arena offsets + advantage) and
 * their handles; *got = mb, or 0 for the reference's nullopt. */
int fm_store_poll(fm_store* s, const char* agent, int64_t version, int64_t mb,
                  const char* prompt_col, const char* response_col, const char* adv_col,
                  fm_sample* samples_out, int64_t* handles_out, int64_t* got);
/* Identity of a polled record (for the reference's MicroBatch view). */
int fm_store_record_id(fm_store* s, const char* agent, int64_t handle, char* input_id_out,
                       size_t cap, int* turns, int* traj, int64_t* version);
/* complete (experience_store.hpp:134-148): NotProcessing unless all polled */
int fm_store_complete(fm_store* s, const char* agent, const int64_t* handles, int64_t n);
/* purge_stale (experience_store.hpp:118-132) */
int fm_store_purge_stale(fm_store* s, const char* agent, int64_t current_version, uint64_t* out);

/* ---- on-device experience table (experience_store.hpp:19-276) --
 * One agent's table kept in the HBM of ctx's GPU: cells (f64 by value, ref
 * columns as token-arena offsets), status flags, processing marks and the
 * canonical key of every record.  The host keeps only the record keys (to
 * raise the reference's synchronous errors: DuplicateSample, RecordNotFound,
 * CellAlreadySet, NotProcessing ...).  The poll's selection, the trainer's
 * micro-batch descriptors, group release (rule_reward + group_advantages) and
 * GPU-generated responses never leave HBM; a poll returns only the chosen slots
 * and the row count the GEMM shapes need.  Records are addressed by the slot
 * insert returns.  Table ops run in call order on the table's own stream, so a
 * poll overlaps the agent's in-flight micro-batch. */
typedef struct fm_dtable fm_dtable;
/* create_table (experience_store.hpp:24-36); capacity = max live records, <= 1<<20 */
int fm_dtable_create(fm_ctx* ctx, const char* agent, const char* const* col_names, const int* col_types,
                     int ncols, int64_t capacity, fm_dtable** out);
int fm_dtable_destroy(fm_dtable* t);
/* insert (experience_store.hpp:44-59), n records of one policy version; all-or-nothing */
int fm_dtable_insert(fm_dtable* t, int64_t version, int n, const char* const* input_ids, const int* turns,
                     const int* trajs, int64_t* slots_out);
/* find (experience_store.hpp:196-201): *slot_out = -1 when absent */
int fm_dtable_find(fm_dtable* t, const char* input_id, int turns, int traj, int64_t version, int64_t* slot_out);
/* set_cell by value (experience_store.hpp:61-80), n cells of one column; all-or-nothing */
int fm_dtable_set_float(fm_dtable* t, const char* column, int n, const int64_t* slots, const double* values);
/* set_cell_payload (experience_store.hpp:82-88): codec bytes ([u64 n][u64 x] * n) into the arena */
int fm_dtable_set_payload(fm_dtable* t, const char* column, int64_t slot, const uint8_t* payload, uint64_t nbytes);
/* Rollout completion on the GPU (rollout.hpp:715-731 with PolicyModel::generate, policy.hpp:119-130)
 * for n records: responses from published f64 weights (dtype 0 or 3) are encoded into the arena
 * and set as `response_col` (+ `logprob_col` as [u64 n][f64] * n, or NULL); prompts/seeds as fm_generate. */
int fm_dtable_generate(fm_dtable* t, const fm_weights* w, const char* response_col, const char* logprob_col,
                       int n, const int64_t* slots, const int32_t* prompts, const int32_t* prompt_off,
                       int max_tokens, const uint64_t* seeds);
/* release_group (rollout.hpp:812-834) for ngroups groups of survivors seg_off[g]..seg_off[g+1]:
 * survivor i's reward = rule_reward(response cell of slot score_slot[i] in tables[score_tab[i]],
 * pattern) (training.hpp:71-83) computed from the arena; advantages = group_advantages(eps)
 * (training.hpp:54-67, bit-identical order); both written to the reward/adv columns of records
 * rec_slot[rec_off[i]..rec_off[i+1]) (tables[rec_tab[.]]).  All tables share one GPU.
 * rewards_out/adv_out (host, one per survivor) may be NULL. */
int fm_dtable_release_groups(fm_dtable* const* tables, int ntables, const char* response_col,
                             const char* reward_col, const char* adv_col, int ngroups, const int32_t* seg_off,
                             const int32_t* score_tab, const int64_t* score_slot, const int32_t* rec_off,
                             const int32_t* rec_tab, const int64_t* rec_slot, const int32_t* pattern,
                             int npattern, double eps, double* rewards_out, double* adv_out);
/* poll_micro_batch (experience_store.hpp:92-114) on the GPU: canonical-first mb (<= 1024) ready
 * records of `version`, marked processing; *got = mb with slots_out in canonical order and
 * *rows_out = their response tokens, or *got = 0 (nullopt).  Column names may be NULL for a
 * selection without trainer descriptors.  *poll_id names the descriptors for fm_train_polled. */
int fm_dtable_poll(fm_dtable* t, int64_t version, int64_t mb, const char* prompt_col,
                   const char* response_col, const char* adv_col, int64_t* slots_out, int64_t* rows_out,
                   int64_t* got, int64_t* poll_id);
/* train_micro_batch (training.hpp:355-430) on a device poll's micro batch: the descriptors
 * are copied D2D from the table's ring (the last 8 polls); same ticket/report as fm_train_micro_batch. */
int fm_train_polled(fm_agent* a, fm_dtable* t, int64_t poll_id, int64_t global_batch, int64_t* ticket_out);
/* complete (experience_store.hpp:134-148): NotProcessing unless every slot is processing */
int fm_dtable_complete(fm_dtable* t, const int64_t* slots, int n);
/* purge_stale (experience_store.hpp:118-132) / purge_inputs (:153-164): device scans */
int fm_dtable_purge_stale(fm_dtable* t, int64_t current_version, uint64_t* out);
int fm_dtable_purge_inputs(fm_dtable* t, const char* const* input_ids, int n, uint64_t* out);
/* drop_record (experience_store.hpp:166-175): *dropped = 0 if absent or processing */
int fm_dtable_drop_record(fm_dtable* t, const char* input_id, int turns, int traj, int64_t version,
                          int* dropped);
/* ready_count (experience_store.hpp:181-187, counted on the GPU) / record_count (:189-191) */
int fm_dtable_ready_count(fm_dtable* t, int64_t version, uint64_t* out);
int fm_dtable_record_count(fm_dtable* t, uint64_t* out);
/* Identity and flags of a slot's record (dump_table view, experience_store.hpp:210-238). */
int fm_dtable_record(fm_dtable* t, int64_t slot, char* input_id_out, size_t cap, int* turns, int* traj,
                     int64_t* version, int* processing, uint32_t* status);
/* Identities of n records at once (the MicroBatch's record copies, experience_store.hpp:111);
 * ids_out holds n strings of id_cap bytes each. */
int fm_dtable_records(fm_dtable* t, int n, const int64_t* slots, char* ids_out, size_t id_cap, int* turns,
                      int* trajs, int64_t* versions);
/* Cells of n slots read back from HBM: by-value columns as f64, ref columns as arena offsets. */
int fm_dtable_read_cells(fm_dtable* t, const char* column, int n, const int64_t* slots, uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
