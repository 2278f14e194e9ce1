/* polycert_b200.h — C-ABI of the B200-native DeepPoly back-substitution
 * verifier (the drop-in boundary for the reference's verifier API).
 *
 * The reference exposes a header-only C++ template API with no FFI
 * (SURVEY.md §8b); the entry points below are exactly the calls a binding of
 * that API needs:
 *
 *   pc_net_create   replaces  validate_model + instantiate<WidenedFloat64>
 *                             (proj/src/model_io.cpp:49-135,
 *                              proj/include/polycert/network.hpp:110-141)
 *   pc_net_test     replaces  verify_robustness(net, box, label, opt)
 *                             (proj/include/polycert/analyzer.hpp:256-276)
 *                             plus analyze(...).state.bounds / .raw
 *                             (analyzer.hpp:171-175, 198-242)
 *   pc_input_box    replaces  input_box<WidenedFloat64>(center, eps, clamp01)
 *                             (network.hpp:160-177)
 *   pc_net_destroy  replaces  ~Network
 *   pc_last_error   carries the message of the reference's exception
 *
 * Plain pointers and sizes only. All arithmetic is the reference's
 * WidenedFloat64 mode (interval.hpp:38-103), reproduced bit-for-bit on the
 * GPU; there is no CPU fallback: without a CUDA device every compute entry
 * point fails with PC_ERR_CUDA.
 */
#ifndef POLYCERT_B200_H
#define POLYCERT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Layer kinds, in the reference's LayerKind order (network.hpp:29). */
enum pc_layer_kind { PC_INPUT = 0, PC_DENSE = 1, PC_CONV = 2, PC_RELU = 3, PC_JOIN = 4 };

/* Status codes: the reference's exception classes map to distinct codes. */
typedef enum {
  PC_OK = 0,
  PC_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (labels, eps, centers) */
  PC_ERR_MODEL = 2,            /* std::runtime_error from validate_model ("model: layer N: ...") */
  PC_ERR_LOGIC = 3,            /* std::logic_error (internal invariants) */
  PC_ERR_CUDA = 4,             /* no device / CUDA failure (no CPU fallback exists) */
  PC_ERR_OOM = 5
} pc_status;

/* One layer, mirroring LayerDoc (network.hpp:34-50). layers[0] must be the
 * input layer. Parameters are FP64 arrays in the reference's flat layouts:
 * dense weights [out][in] row-major (network.hpp:94); conv filter
 * ((fy*fw+fx)*cin+ci)*cout+co (network.hpp:43). */
typedef struct {
  int kind;      /* pc_layer_kind */
  int n_preds;   /* 0 input, 2 join, else 1 */
  int preds[2];
  int n_out;     /* dense: number of rows */
  int fw, fh, sw, sh, pw, ph, cin, cout; /* conv */
  const double* weights; /* dense weights or conv filter */
  const double* bias;    /* dense: n_out, conv: cout */
} pc_layer_desc;

/* AnalysisOptions (analyzer.hpp:164-169). memory_budget bounds the device
 * workspace of one pass (0: default); results are chunk-invariant.
 * exec_mode: the host-driven schedule launches each step from the host and
 * reads every checkpoint's surviving-row count (exact grids, chunking, early
 * exit); the device-driven one keeps the live-row count on the device, so a
 * whole verification is captured once as a CUDA graph and replayed per image
 * (needs every pass in one chunk; launches are sized for all of a layer's
 * neurons). auto = host-driven. Results identical. */
typedef struct {
  int early_term;          /* default 1 */
  long long chunk_rows;    /* 0: derive from memory_budget */
  long long memory_budget; /* bytes; 0: engine default */
  int device;              /* CUDA ordinal; -1: current */
  int exec_mode;           /* 0 auto, 1 host-driven schedule, 2 device-driven (CUDA graph) */
  int numeric_mode;        /* 0 the reference's WidenedFloat64, bit for bit (default);
                              1 fast: native directed rounding (RD / RU FMAs and adds) in
                              the conv coefficients, the constant chains and the
                              concretisations — sound (outward), not bit-identical */
} pc_options;

/* PassStats (backsub.hpp:119-136). */
typedef struct {
  long long rows_total;
  long long rows_terminated_early;
  long long gbc_madds;
  long long gbc_dense_equiv;
  long long dense_madds;
  long long checkpoints;
} pc_stats;

typedef struct pc_net pc_net;

void pc_default_options(pc_options* opt);

/* Validation only (model_io.cpp:49-135), no device needed. out_shapes
 * (optional) receives n_layers x {w, h, c}. */
pc_status pc_validate(const pc_layer_desc* layers, int n_layers, int in_w, int in_h, int in_c,
                      int* out_shapes);

/* Validate + upload. Error messages match validate_model's. */
pc_status pc_net_create(const pc_layer_desc* layers, int n_layers, int in_w, int in_h, int in_c,
                        const pc_options* opt, pc_net** out);
void pc_net_destroy(pc_net* net);

int pc_net_num_layers(const pc_net* net);
/* Neurons in layer k (numel of its output shape); -1 if out of range. */
long long pc_net_layer_numel(const pc_net* net, int k);
long long pc_net_total_neurons(const pc_net* net);
int pc_net_output_size(const pc_net* net);

/* Widened input region (network.hpp:160-177). HOST arrays of n values. */
pc_status pc_input_box(const double* center, int n, double eps, int clamp01, double* lo, double* up);

/* test(lo, up, label): HOST input box (n = input numel) in, verdict out.
 * label < 0 runs the analysis only (no margin pass). margins: n_out-1
 * certified lower bounds of out_label - out_j, ascending j != label.
 * bounds_* (optional, may be NULL): padded per-neuron bounds concatenated
 * over layers in id order; raw_* the unpadded freeze-test twin. */
pc_status pc_net_test(pc_net* net, const double* lo, const double* up, int label, int* verified,
                      double* margins, double* bounds_lo, double* bounds_hi, double* raw_lo,
                      double* raw_hi, pc_stats* stats);

/* pc_net_test with per-call options: the AnalysisOptions of this one
 * verify_robustness / analyze call (early_term, chunk_rows, memory_budget,
 * exec_mode; `device` is ignored: the net's device is used). NULL: the net's
 * options. Lets one pc_net (the device weights) serve calls with different
 * options concurrently, as the reference's immutable Network does
 * (analyzer.hpp:198-276, AnalysisOptions analyzer.hpp:164-169). */
pc_status pc_net_test_ex(pc_net* net, const pc_options* call_opt, const double* lo,
                         const double* up, int label, int* verified, double* margins,
                         double* bounds_lo, double* bounds_hi, double* raw_lo, double* raw_hi,
                         pc_stats* stats);

/* Same with the input box already resident in device memory (d_lo, d_up are
 * CUDA device pointers on the net's device); outputs are host arrays. */
pc_status pc_net_test_device(pc_net* net, const double* d_lo, const double* d_up, int label,
                             int* verified, double* margins, pc_stats* stats);

/* Candidate label: unique argmax of the concrete forward pass at `center`
 * (forward_eval, eval.hpp:39-102; unique_argmax, tools/main.cpp:86-100), -1
 * on a tie. logits (optional) receives the n_out outputs. HOST arrays. */
pc_status pc_net_candidate(pc_net* net, const double* center, int* label, double* logits);

/* The CUDA stream (cudaStream_t) every kernel of this net is launched on,
 * for callers that time or order work around pc_net_test* with CUDA events. */
void* pc_net_stream(const pc_net* net);

/* Throughput entry: verify n_images boxes concurrently, `concurrency` host
 * worker threads each driving its own stream and per-call state on the net's
 * device (images are independent; results equal pc_net_test's).
 * lo/up: n_images x input-numel, HOST arrays (device arrays if
 * device_inputs != 0). labels[i] < 0: analysis only. verified[n_images],
 * margins[n_images x (n_out-1)], stats[n_images] are optional outputs.
 * device_ms (optional): device time of the whole batch, CUDA events on a
 * master stream every worker stream waits on / is awaited by. */
pc_status pc_net_test_batch(pc_net* net, int n_images, const double* lo, const double* up,
                            int device_inputs, const int* labels, int concurrency, int* verified,
                            double* margins, pc_stats* stats, double* device_ms);

/* Row sharding across ranks (one process per GPU). With
 * world > 1 every rank runs every pass's seed and refresh (identical,
 * deterministic), back-substitutes only its contiguous slice of the pass's
 * live rows (and of the margin rows), and the refined candidate bounds
 * (32 B per row; 8 B per margin row) are all-gathered before the write-back —
 * the path's one exchange step. Results are bit-identical to world = 1.
 * `allgather` must gather `bytes` from every rank's device buffer d_send into
 * d_recv (rank-major, world * bytes), ordered on `stream` (a cudaStream_t),
 * e.g. ncclAllGather(d_send, d_recv, bytes, ncclUint8, comm, stream); it
 * returns 0 on success. Every rank must call pc_net_test on the same box and
 * label. pc_net_test_batch refuses a sharded net. world = 1 disables. */
typedef int (*pc_allgather_fn)(void* user, const void* d_send, void* d_recv, size_t bytes,
                               void* stream);
pc_status pc_net_set_sharding(pc_net* net, int rank, int world, pc_allgather_fn allgather,
                              void* user);

/* Native NCCL transport for row sharding (no host callback on the data
 * path): rank 0 creates a 128-byte id with pc_nccl_unique_id and shares it
 * out of band (e.g. torch.distributed broadcast); every rank creates its
 * communicator on the net's device with pc_nccl_comm_create and passes
 * pc_nccl_allgather with the communicator as `user` to pc_net_set_sharding:
 * the exchange is then one ncclAllGather on the engine's stream. libnccl.so.2
 * is loaded at run time (dlopen). Return 0 / non-NULL on success; `err`
 * receives the message otherwise. */
typedef struct pc_nccl_comm pc_nccl_comm;
int pc_nccl_unique_id(void* out128, char* err, int err_len);
pc_nccl_comm* pc_nccl_comm_create(int device, int rank, int world, const void* id128, char* err,
                                  int err_len);
void pc_nccl_comm_destroy(pc_nccl_comm* comm);
int pc_nccl_allgather(void* user, const void* d_send, void* d_recv, size_t bytes, void* stream);

/* Kernel launches issued by this thread's last pc_net_test* call. */
long long pc_last_launch_count(void);

/* Device timing of the last call: total milliseconds measured with CUDA
 * events on the engine stream, and the milliseconds spent in the dense
 * back-substitution kernel (the roofline kernel) with its algorithmic bytes. */
void pc_last_timing(double* total_ms, double* dense_kernel_ms, double* dense_kernel_bytes,
                    long long* dense_kernel_launches);
/* The same for one back-substitution coefficient kernel of the last
 * pc_net_test* call on this thread: kernel 0 = the dense kernel
 * (k_dense_coef*), 1 = the conv kernel (k_gbc_live / k_gbc_sparse2 / k_gbc_coef): summed
 * CUDA-event milliseconds over its launches (on the stream each is launched
 * on), algorithmic bytes (coefficient rows in and out, 16 B per interval,
 * plus the weights / filter once per launch) and the launch count. */
void pc_last_kernel_timing(int kernel, double* ms, double* bytes, long long* launches);

/* Interval multiply-adds the live-cell conv kernel (k_gbc_live) executed in
 * the last pc_net_test* call on this thread (device-counted; the reference's
 * PassStats.gbc_madds also counts the cells whose value no result reads). */
double pc_last_conv_executed_madds(void);

/* Timing mode: serial != 0 runs every walk on one stream and one pipeline,
 * so the per-launch CUDA events of pc_last_kernel_timing time each kernel
 * alone (roofline measurement); results are identical. Not thread-safe
 * against concurrent pc_net_test* calls on the net. */
pc_status pc_net_set_serial(pc_net* net, int serial);

/* Measured FP64 FMA throughput of the device (FMA/s): a register-resident
 * DFMA kernel (8 independent chains per thread, every SM), timed with CUDA
 * events; the FP64-pipe roofline denominator. */
pc_status pc_fp64_peak(int device, double* fma_per_s);

/* Interval multiply-adds the dense-kernel launches of the last call executed
 * (rows x live predecessor cells x nonzero frame cells walked, summed over
 * launches; device-counted, all worker contexts of a batch). */
double pc_last_dense_madds(void);

/* Per-kernel-class device time of this thread's last pc_net_test* call as a
 * JSON object {class: [launches, ms]} (collected only when the environment
 * variable PC_PROFILE=1 is set when the net is created). Returns the length. */
int pc_last_profile(char* buf, int len);

/* Numeric-core self test (device): out[i] = op(a[i], b[i]) with op 0
 * add_down, 1 add_up, 2 mul_down, 3 mul_up, 4 div_down, 5 div_up,
 * 6 ulp_above(a) (interval.hpp:59-102); 7/8 the direction-generic chain add
 * (up/down); 9/10 nextafter(a, +/-inf); 11/12 the compare-free band product
 * (down/up) and 13/14 band sum (down/up) used by the conv/dense kernels when
 * their operands are proven in band. HOST arrays. */
pc_status pc_scalar_ops(int op, const double* a, const double* b, double* out, long long n);

/* Chain-fold self test (device): out[c] = acc0[c] folded with terms[c*len ..
 * c*len+len) in order by add_up (up[c] & 1) or add_down (interval.hpp:59-68),
 * NaN terms skipped — the row-constant / concretisation chains of
 * backsub.hpp:365-389, 740-760, evaluated by the warp-scan fold the chain
 * kernels use (csrc/scanfold.cuh; up[c] & 2: its 32-link variant; & 8: its
 * prefetching variant over a term array; up[0] & 4: the CTA-wide fold for every
 * chain, & 16 with it: the CTA-wide fold with local retry). HOST arrays. */
/* Chain-fold diagnostics of the current device: out4 (optional, 8 entries)
 * receives the counters since the last call — scan steps, links committed by
 * scans, scalar links after a failed step, frame-less scalar links, rounding
 * ties met, out-of-range terms met, failed links that grew past / shrank or
 * flipped out of the accumulator's binade (prefetching fold) — which are then
 * reset; on != 0 enables counting (off by default). */
pc_status pc_scan_stats(int on, unsigned long long* out4);

pc_status pc_chain_fold(int n_chains, int len, const double* acc0, const double* terms, const int* up,
                        double* out);

const char* pc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* POLYCERT_B200_H */
