/*
 * ds2ctc.h -- C-ABI of the B200-native Deep Speech 2 CTC loss + gradient.
 *
 * Drop-in boundary for the reference's CTC entry point
 *   asr::ctc::ctc_loss_reference(const Matrix& frame_logits,
 *                                const std::vector<int>& label, int blank)
 *   (/root/reference/proj/include/asr/ctc.hpp:84-87, proj/src/ctc.cpp:171-207)
 * as the trainer drives it, one utterance at a time, inside
 *   asr::trainer::train_epoch (proj/src/trainer.cpp:155-171)
 * and, cost-only, inside evaluate_mean_loss (trainer.cpp:201-214).
 *
 * The reference has no batched API; this header defines the batched,
 * warp-ctc-style boundary that SURVEY.md §8b specifies. Its contract is
 * per-utterance equivalence with ctc_loss_reference on the slice
 * X[0:T_b, b, :] widened to fp64:
 *
 *   costs[b]          = ctc_loss_reference(...).loss           (fp32; +inf if infeasible)
 *   gradients[t][b][:] = ctc_loss_reference(...).logit_grad(t,:) for t < T_b,
 *                        0 for T_b <= t < T_max, and all-zero rows for an
 *                        infeasible utterance (the trainer's convention,
 *                        trainer.cpp:160-166).
 *
 * Tolerance: |cost - ref| / |ref| <= 1e-4 and max |grad - ref| <= 1e-4 (fp32
 * outputs vs the fp64 reference). The summation order differs from the
 * reference (linear-space occupancy sums instead of log-space folds,
 * ctc.cpp:76; log p from the alpha/beta meet point instead of the last alpha
 * column, ctc.cpp:188) -- see DESIGN.md §Numerics.
 *
 * All entry points are thread-safe across distinct (device, stream, workspace).
 * No exceptions cross the ABI; errors are status codes.
 */
#ifndef DS2CTC_H
#define DS2CTC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DS2CTC_STATUS_SUCCESS = 0,
  DS2CTC_STATUS_INVALID_VALUE = 1,   /* bad shape/length/label/blank, or workspace too small */
  DS2CTC_STATUS_EXECUTION_FAILED = 2,/* CUDA launch / runtime error */
  DS2CTC_STATUS_MEMOPS_FAILED = 3,   /* host<->device copy or allocation failure */
  DS2CTC_STATUS_UNSUPPORTED = 4      /* e.g. 2L+1 > DS2CTC_MAX_STATES, or no sm_100 device */
} ds2ctc_status;

/* Largest blank-extended label (2L+1) one utterance may have. */
#define DS2CTC_MAX_STATES 4095

/* Human-readable status. Replaces the reference's exception messages
 * ("asr: ...", proj/include/asr/common.hpp:37-44). */
const char* ds2ctc_status_string(ds2ctc_status status);

/* Library version string ("ds2ctc <semver> sm_100a"). */
const char* ds2ctc_version(void);

/*
 * Device workspace needed by ds2ctc_compute_loss for this batch shape.
 * label_lengths / input_lengths are HOST arrays [minibatch]. alphabet_size
 * INCLUDES the blank (A = reference alphabet_size + 1, network.cpp:135).
 * Replaces the reference's per-call Matrix allocations (ctc.cpp:175,181,197,
 * the KeyGroups of ctc.cpp:195): the caller owns all memory.
 */
ds2ctc_status ds2ctc_get_workspace_size(const int* label_lengths, const int* input_lengths, int alphabet_size,
                                        int minibatch, size_t* bytes);

/*
 * CTC loss and gradient for a batch.
 *   activations   DEVICE fp32 [T_max][minibatch][alphabet_size], pre-softmax logits,
 *                 T_max = max(input_lengths). Softmax is applied internally
 *                 (ctc.hpp:37-40), so logits and log-probabilities are interchangeable.
 *   gradients     DEVICE fp32, same shape, or NULL for cost only (evaluate_mean_loss,
 *                 trainer.cpp:201-214; datapipe.cpp:99). Gradient w.r.t. the
 *                 pre-softmax activations (ctc.cpp:69-79).
 *   flat_labels   HOST int32, concatenation of the minibatch labels (sum(label_lengths)).
 *   label_lengths HOST int32 [minibatch].
 *   input_lengths HOST int32 [minibatch], each in [0, T_max].
 *   blank_label   index of the blank in [0, alphabet_size); the trainer uses
 *                 alphabet_size - 1 (trainer.cpp:127).
 *   costs         DEVICE fp32 [minibatch] (-log p, +inf when infeasible).
 *   workspace     DEVICE, at least ds2ctc_get_workspace_size() bytes, 256-byte aligned.
 *   stream        cudaStream_t (NULL = legacy default stream). Asynchronous.
 *                 A variable-length batch (B >= 256, alphabet <= 128, labels
 *                 spread by length) may run as length-split sub-batches on
 *                 library streams forked from and joined back into `stream`
 *                 (DS2CTC_LENGTH_SPLIT=0 disables); ordering w.r.t. `stream`
 *                 is unchanged, and the workspace query accounts for it.
 * minibatch == 0 is a valid no-op (an empty data-parallel shard, trainer.cpp:141-155).
 */
ds2ctc_status ds2ctc_compute_loss(const float* activations, float* gradients, const int* flat_labels,
                                  const int* label_lengths, const int* input_lengths, int alphabet_size,
                                  int minibatch, int blank_label, float* costs, void* workspace, void* stream);

/* Same as ds2ctc_compute_loss, but checks the workspace size explicitly. */
ds2ctc_status ds2ctc_compute_loss_checked(const float* activations, float* gradients, const int* flat_labels,
                                          const int* label_lengths, const int* input_lengths, int alphabet_size,
                                          int minibatch, int blank_label, float* costs, void* workspace,
                                          size_t workspace_bytes, void* stream);

/*
 * Host-buffer entry point: the reference-facing call (the reference takes and
 * returns host matrices). activations / gradients / costs are HOST arrays in
 * the layout above (pinned memory gives full PCIe bandwidth); the library
 * copies them through a per-thread device context on `device`, runs the same
 * kernels, copies the results back and synchronises before returning.
 */
ds2ctc_status ds2ctc_compute_loss_host(const float* activations, float* gradients, const int* flat_labels,
                                       const int* label_lengths, const int* input_lengths, int alphabet_size,
                                       int minibatch, int blank_label, float* costs, int device);

/*
 * CTC forced alignment, the batched device counterpart of
 *   std::vector<int> viterbi_align(const Matrix& frame_logprobs,
 *                                  const std::vector<int>& label, int blank)
 * (proj/include/asr/ctc.hpp:97-101, proj/src/ctc.cpp:327-370), used by
 * datapipe::align_frames / segment (datapipe.cpp:27-92) and `asr align`.
 * For each b: the highest-probability lattice path of X[0:T_b, b, :] whose
 * collapse is the label, ties resolved exactly as the reference (stay >
 * advance > skip; terminal blank unless the terminal label is strictly
 * better). alignments is DEVICE int32 [minibatch][T_max] (T_max = max T_b):
 * the frame symbols, -1 past T_b. status is DEVICE int32 [minibatch]: 0 =
 * aligned, 1 = no alignment (T_b < min_frames, T_b == 0, or every path has
 * zero probability -- where the reference throws; the row is all -1).
 * activations as ds2ctc_compute_loss; labels and lengths are host arrays.
 * Asynchronous on `stream`; the workspace comes from
 * ds2ctc_viterbi_get_workspace_size (per-utterance backpointers).
 */
ds2ctc_status ds2ctc_viterbi_get_workspace_size(const int* label_lengths, const int* input_lengths,
                                                int alphabet_size, int minibatch, size_t* bytes);
ds2ctc_status ds2ctc_viterbi_align(const float* activations, const int* flat_labels, const int* label_lengths,
                                   const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                   int* alignments, int* status, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* Host-buffer form of ds2ctc_viterbi_align (alignments [minibatch][T_max],
 * status [minibatch] are HOST arrays); synchronous, on `device`. */
ds2ctc_status ds2ctc_viterbi_align_host(const float* activations, const int* flat_labels, const int* label_lengths,
                                        const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                        int* alignments, int* status, int device);

/*
 * Full CTC lattice export, the batched device counterpart
 * of CtcLattice ctc_lattice(const Matrix& frame_logits, const std::vector<int>&
 * label, int blank) (proj/include/asr/ctc.hpp:55-60,68-71; ctc.cpp:145-169):
 * fp64 natural-log alpha and emission-exclusive beta of every lattice cell
 * and log p, computed operation by operation as the reference (debug /
 * verification path of the column-parallel scheme). ds2ctc_lattice_get_sizes
 * gives the cell count (sum_b (2 L_b + 1) T_b) of alpha and of beta, and the
 * workspace bytes. alpha / beta are DEVICE fp64 [cells]: utterance b's block
 * starts at sum_{b'<b} (2 L_b' + 1) T_b' and is row-major [2 L_b + 1][T_b]
 * (the reference Matrix (s, t)); log_prob is DEVICE fp64 [minibatch] (-inf
 * when no path has nonzero probability). Every T_b must be >= 1 (the
 * reference throws, ctc.cpp:146): INVALID_VALUE otherwise.
 */
ds2ctc_status ds2ctc_lattice_get_sizes(const int* label_lengths, const int* input_lengths, int minibatch,
                                       size_t* cells, size_t* workspace_bytes);
ds2ctc_status ds2ctc_ctc_lattice(const float* activations, const int* flat_labels, const int* label_lengths,
                                 const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                 double* alpha, double* beta, double* log_prob, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* Host-buffer form of ds2ctc_ctc_lattice (alpha, beta [cells], log_prob
 * [minibatch] are HOST arrays); synchronous, on `device`. */
ds2ctc_status ds2ctc_ctc_lattice_host(const float* activations, const int* flat_labels, const int* label_lengths,
                                      const int* input_lengths, int alphabet_size, int minibatch, int blank_label,
                                      double* alpha, double* beta, double* log_prob, int device);

/*
 * Per-shard {sum of feasible costs, number of infeasible utterances} as fp64
 * (infeasible = cost +inf; a NaN cost is feasible, as in the reference, and
 * makes the sum NaN)
 * [2] on the device, the two scalars train_epoch accumulates
 * (local_loss / local_skipped, trainer.cpp:160-168) and all-reduces
 * (trainer.cpp:176-179). Fixed summation order (deterministic). costs and
 * out2 are DEVICE pointers; asynchronous on `stream`.
 */
ds2ctc_status ds2ctc_loss_sum(const float* costs, int minibatch, double* out2, void* stream);

/*
 * The same per-shard sums fused with their all-reduce over NVLink peer memory
 * (trainer.cpp:176-179; allreduce.cpp:301-341 with its fixed fold order):
 * one single-warp kernel per rank stores its pair into every rank's mailbox
 * and folds all `world` pairs in rank order into out2 (DEVICE fp64 [2]),
 * bitwise identical on every rank. Setup, once per process group:
 * ds2ctc_mailbox_alloc gives this rank's mailbox and a 64-byte CUDA IPC
 * handle to exchange (e.g. torch.distributed.all_gather_object);
 * ds2ctc_mailbox_open maps each peer's handle. peer_mailboxes[r] is rank r's
 * mailbox as seen by this process (its own pointer for r == rank). `seq`
 * starts at 1 and increases by one per call on every rank. Asynchronous on
 * `stream`; world <= 8.
 */
ds2ctc_status ds2ctc_mailbox_alloc(int world, void** mailbox, void* ipc_handle);
ds2ctc_status ds2ctc_mailbox_open(const void* ipc_handle, void** peer_mailbox);
ds2ctc_status ds2ctc_mailbox_close(void* peer_mailbox, int own);
ds2ctc_status ds2ctc_loss_sum_allreduce(const float* costs, int minibatch, double* out2, void* const* peer_mailboxes,
                                        int rank, int world, unsigned long long seq, void* stream);
/*
 * Parameter-gradient all-reduce over NVLink peer memory (trainer.cpp:175:
 * ring_allreduce of the gradients, allreduce.cpp:301-341): every rank's
 * data[n] (fp32, device) becomes the sum over ranks folded in rank order
 * (allreduce.hpp:91-95) -- bitwise identical on every rank and run to run.
 * Setup once per rank: ds2ctc_exchange_size(n) bytes from
 * ds2ctc_exchange_alloc (zeroed; 64-byte CUDA IPC handle out), the peers'
 * regions mapped with ds2ctc_mailbox_open, released with ds2ctc_mailbox_close.
 * Every rank calls with the same n, its rank, world (<= 8) and the same seq
 * (1, 2, 3, ... per call). One kernel: each CTA stages its slice, publishes
 * a per-slice flag to every rank, waits for every rank's flag (at most 20 s;
 * on timeout the slice is NaN and ds2ctc_reduce_fault reports seq), folds.
 */
ds2ctc_status ds2ctc_exchange_size(size_t n, size_t* bytes);
ds2ctc_status ds2ctc_exchange_alloc(size_t bytes, void** region, void* ipc_handle);
ds2ctc_status ds2ctc_vec_allreduce(float* data, size_t n, void* const* peer_regions, int rank, int world,
                                   unsigned long long seq, void* stream);

/*
 * Lost-peer check of ds2ctc_loss_sum_allreduce. Each call waits at most 20 s
 * (%globaltimer) for the peers' pairs of its step; on timeout it writes NaN
 * into out2 (never a stale fold) and records the step. This reads (after
 * the recorded kernels finished: it synchronises with the device's legacy
 * stream) and clears the first timed-out `seq`, 0 if none. After a timeout
 * the mailboxes must be closed and re-created on every rank.
 */
ds2ctc_status ds2ctc_reduce_fault(unsigned long long* seq);

/*
 * Stage timing for benchmarks: when enabled for the calling thread with
 * `slots` > 0, each compute call records CUDA events on its stream around
 * every kernel of the pipeline into the next of `slots` event sets (no host
 * synchronisation). ds2ctc_profile_read(i) synchronises on call i (counted
 * from the enable, i < slots) and writes ms[4] = {pair kernel (alpha||beta
 * chain, fused gradient), dense gradient pass (large alphabets: k_dense after
 * the pair kernel; with DS2CTC_DENSE_OVERLAP=1 the softmax pass alone, which
 * then runs concurrently with the pair kernel), cost finalisation, whole
 * call}. slots == 0 disables.
 */
ds2ctc_status ds2ctc_profile_enable(int slots);
ds2ctc_status ds2ctc_profile_read(int call_index, float* ms);

/*
 * Diagnostics: every inter-warp wait inside the pair kernel is bounded; a
 * wait that exceeds its bound (a protocol bug) is recorded instead of hanging
 * the GPU. Synchronises the device, writes {kind, block, warp, step} of the
 * first such event since the last call (all zero if none) and clears it.
 */
ds2ctc_status ds2ctc_debug_watchdog(unsigned long long* out4);

/*
 * The CTC gradient's consumer: the output fully connected
 * layer's backward pass, FullyConnectedLayer::backward (proj/src/nn.cpp:874-899)
 * for the output layer built by network.cpp:135 (no ReLU, no batch norm), on
 * tcgen05 tensor cores (tf32 inputs, fp32 accumulation) with the gradient
 * still on the device:
 *   db[A]    += sum_r dlogits[r][:]          (nn.cpp:886-890)
 *   dw[A][H] += dlogits^T x                  (matmul_tn, nn.cpp:894)
 *   dx[r][H]  = dlogits w                    (matmul, nn.cpp:895)
 * dlogits is DEVICE fp32 [rows][out_dim] -- the gradients buffer of
 * ds2ctc_compute_loss viewed as rows = T_max * minibatch (padded frames are
 * zero rows); x DEVICE fp32 [rows][in_dim] (the layer's input, same row
 * order); w DEVICE fp32 [out_dim][in_dim]; dw / db accumulate (the caller
 * zeroes them per step, like zero_grads, trainer.cpp:152); dx is written;
 * dw, db, dx are each nullable. in_dim must be a multiple of 4 and the
 * buffers 16-byte aligned (TMA). The workspace (ds2ctc_fc_backward_workspace_size)
 * re-pitches the gradient rows when out_dim % 4 != 0. Asynchronous on `stream`.
 * Tolerance vs the fp64 reference: tf32 products (10-bit mantissa), fp32 sums.
 */
ds2ctc_status ds2ctc_fc_backward_workspace_size(int rows, int out_dim, int in_dim, size_t* bytes);
ds2ctc_status ds2ctc_fc_backward(const float* dlogits, const float* x, const float* w, float* dw, float* db, float* dx,
                                 int rows, int out_dim, int in_dim, void* workspace, size_t workspace_bytes,
                                 void* stream);
/* ---------------------------------------------------------------------
 * H1 host scheduler (trainer.cpp:58-91, 140-143) -- pure host functions.
 * ------------------------------------------------------------------- */

/* SortaGrad visiting order, identical to asr::trainer::sortagrad_order
 * (trainer.cpp:58-91): epoch 0 stable-sorts by length; later epochs shuffle
 * whole minibatches with Rng(seed*0x9e3779b9 + epoch + 1). out_order[n]. */
ds2ctc_status ds2ctc_sortagrad_order(const int* lengths, int n, int global_batch, int epoch, uint64_t seed,
                                     int sortagrad_on, int64_t* out_order);

/* The reference's contiguous rank slice of one global minibatch
 * (trainer.cpp:140-143): [*begin, *end) positions within the batch. */
ds2ctc_status ds2ctc_rank_slice(int batch_n, int minibatch_size, int rank, int* begin, int* end);

/*
 * Length-aware re-deal of one global minibatch across `world` GPUs:
 * longest-processing-time-first on the estimated cost of each utterance,
 * T_b * (1 + alphabet/1024) (serial chain ~ T_b frames, HBM ~ T_b * alphabet
 * bytes; ties broken by label length). out_rank[n] receives the rank
 * of each utterance; ranks keep the batch's SortaGrad composition, and the
 * per-utterance results are order-independent, so parity is unaffected.
 * out_load (nullable, [world]) receives each rank's estimated cost.
 */
ds2ctc_status ds2ctc_shard_lpt(const int* input_lengths, const int* label_lengths, int n, int alphabet_size,
                               int world, int* out_rank, double* out_load);

#ifdef __cplusplus
}
#endif

#endif /* DS2CTC_H */
