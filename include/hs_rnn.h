/*
 * hs_rnn.h — C ABI of the B200-native RNN DAG executor (libhsrnn.so).
 *
 * This is the seam under the reference's Python API.  The reference
 * (`hetsched`) has no FFI: its executor is the virtual-time replay
 * `engine.simulate` (/root/reference/pkg/src/hetsched/engine.py:265-418) and its
 * profiler the seeded generator `synth_profile` (costmodel.py:176-221).  The
 * entry points below replace those two seams with real B200 execution and
 * timing; the Python wrapper (paper_2307_11339_b200/rnn.py) binds them with
 * ctypes exactly as INTEGRATION.md shows.
 *
 *   reference seam                               replaced by
 *   engine.simulate(graph, cm, plan) -> Trace    hs_rnn_forward / hs_rnn_forward_packed
 *                                                (whole DAG, all-GPU plan segments)
 *   engine.simulate, per-node NodeSpan           hs_rnn_run_cells (one layer-direction,
 *                                                a contiguous run of timesteps = a GPU
 *                                                segment of a hybrid plan)
 *   costmodel.synth_profile -> W[:,0]            hs_rnn_profile_cells (per-cell ms from
 *                                                per-step %globaltimer stamps), and the
 *                                                per-layer CUDA-event times of
 *                                                hs_rnn_forward_packed(..., layer_ms)
 *
 * Conventions: every pointer argument that names a tensor is a DEVICE pointer
 * allocated by the caller (PyTorch); the library never allocates or frees
 * caller memory and keeps no state between calls apart from per-device
 * attribute caches.  `stream` is a cudaStream_t passed as void*.  Returns
 * HS_OK (0) or an HS_ERR_* code; hs_last_error() gives a thread-local message.
 * No C++ exception crosses this boundary.  There is no CPU fallback: on a host
 * without a usable sm_100 device every compute entry point fails.
 *
 * Tensor layouts (PyTorch nn.LSTM / nn.GRU, batch_first=False):
 *   x      [T, B, I]             fp32
 *   y      [T, B, dirs*H]        fp32
 *   h0,hn  [layers*dirs, B, H]   fp32 (h0/c0 may be NULL = zeros)
 *   c0,cn  [layers*dirs, B, H]   fp32 (LSTM only; NULL for GRU)
 *   per layer-direction ld = l*dirs + d:
 *     w_ih[ld] [G*H, I_l], w_hh[ld] [G*H, H], b_ih[ld] [G*H], b_hh[ld] [G*H]
 *     I_0 = input, I_l = dirs*H for l >= 1; G = 4 (LSTM i,f,g,o) or 3 (GRU r,z,n)
 */
#ifndef HS_RNN_H
#define HS_RNN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HS_RNN_ABI_VERSION 1

enum hs_cell { HS_CELL_LSTM = 0, HS_CELL_GRU = 1 };
enum hs_dtype { HS_DTYPE_F32 = 0, HS_DTYPE_BF16 = 1 };
enum hs_algo {
  HS_ALGO_AUTO = 0,   /* pick the fastest path that supports the shape        */
  HS_ALGO_SIMT = 1,   /* FP32 FFMA kernels (any shape; reference for the TC path) */
  HS_ALGO_TC = 2      /* tcgen05 tensor-core kernels (split-bf16 in f32 mode)  */
};
enum hs_status {
  HS_OK = 0,
  HS_ERR_INVALID = 1,     /* bad descriptor / argument                      */
  HS_ERR_CUDA = 2,        /* a CUDA runtime call failed                       */
  HS_ERR_UNSUPPORTED = 3, /* shape/dtype/algo combination not implemented     */
  HS_ERR_WORKSPACE = 4,   /* workspace or packed buffer too small             */
  HS_ERR_NO_DEVICE = 5    /* no sm_100 device visible                         */
};

typedef struct hs_rnn_desc {
  int32_t cell;    /* hs_cell */
  int32_t layers;  /* L >= 1 */
  int32_t dirs;    /* 1 or 2 */
  int32_t input;   /* I (layer-0 input size) */
  int32_t hidden;  /* H */
  int32_t seq;     /* T */
  int32_t batch;   /* B */
  int32_t dtype;   /* hs_dtype: F32 = fp32-exact (max-abs 1e-4), BF16 = opt-in */
  int32_t algo;    /* hs_algo */
  int32_t upload_chunks;  /* hs_rnn_forward_host: time chunks x is uploaded in (0 = 4).
                            1 suits request streams (x already uploaded during the
                            previous request); more chunks lower single-request latency */
  int32_t async_outputs;  /* hs_rnn_forward_host: 1 = the D2H copies of y / h_n / c_n are NOT
                            joined into `stream`: the next request's compute may start while
                            they drain; hs_rnn_outputs_ready() waits for them.  0 = all work,
                            copies included, complete when `stream` reaches the call's end */
  int32_t reserved[5];
} hs_rnn_desc;

/* ABI version of the loaded library (HS_RNN_ABI_VERSION). */
int hs_abi_version(void);

/* Thread-local description of the last failure in this thread. */
const char* hs_last_error(void);

/* Kernels launched by the last hs_rnn_forward_packed / hs_rnn_forward_host /
 * hs_rnn_run_cells call on this thread (memsets and copies excluded). */
int hs_rnn_last_launch_count(void);

/* Which algorithm hs_rnn_forward_packed would run for this descriptor
 * (HS_ALGO_SIMT or HS_ALGO_TC) on the current device. */
int hs_rnn_resolve_algo(const hs_rnn_desc* desc, int32_t* algo);

/* Execution plan the library picks for this descriptor (static device
 * limits), 8 ints: [0] algo (HS_ALGO_*), [1] tensor-core K-split cluster size
 * S, or the small-shape kernel's cluster size C (SIMT), [2] W_hh ring depth
 * (0 = W_hh resident in shared memory, > 0 = streamed from L2 every step),
 * [3] batch slices, [4] 1 if the small-shape cluster kernel runs, [5] 1 if the
 * layers run as one single-GPU layer wavefront (every layer's recurrence and
 * input projection in one launch; [1] is then its K-split), [6] the wave's
 * CTAs per SM (1 or 2), [7] 0. */
int hs_rnn_plan(const hs_rnn_desc* desc, int32_t* info);

/* Bytes of device workspace needed by hs_rnn_forward_packed / run_cells. */
int hs_rnn_workspace(const hs_rnn_desc* desc, size_t* bytes);

/* Bytes of the packed (kernel-layout) weight buffer. */
int hs_rnn_packed_size(const hs_rnn_desc* desc, size_t* bytes);

/* Repack PyTorch-layout weights (arrays of layers*dirs device pointers) into
 * the kernel layout (bias folding, unit-block tiling, split-bf16 planes). */
int hs_rnn_pack_weights(const hs_rnn_desc* desc,
                        const void* const* w_ih, const void* const* w_hh,
                        const void* const* b_ih, const void* const* b_hh,
                        void* packed, size_t packed_bytes, void* stream);

/* Whole-DAG forward with packed weights.  If `layer_ms` is non-NULL it must
 * hold 2*layers floats: per layer, the input-projection GEMM time and the
 * recurrent-wavefront time in ms (CUDA events; the call then synchronizes). */
int hs_rnn_forward_packed(const hs_rnn_desc* desc, const void* packed,
                          const void* x, const void* h0, const void* c0,
                          void* y, void* hn, void* cn,
                          void* workspace, size_t ws_bytes, void* stream,
                          float* layer_ms);

/* Per-cell GPU cost of the whole-DAG forward (the measured replacement of
 * costmodel.synth_profile's W[:, 0], costmodel.py:176-221, which the planner
 * reads per node, costmodel.py:141-150).  Runs hs_rnn_forward_packed once with
 * per-step %globaltimer stamps in each layer-direction's recurrence and
 * synchronizes.  cell_ms [layers*dirs*T] is indexed like the cell grid's nodes,
 * (l*dirs + d)*T + t (graph.gen_lstm_grid / gen_bilstm_grid): each cell gets
 * its measured step period, scaled so that all cells sum to the measured
 * forward (CUDA events; also returned in *forward_ms when non-NULL).  Paths
 * without stamps (SIMT, small-shape cluster kernel) get the mean period.
 * Needs the workspace of hs_rnn_workspace. */
int hs_rnn_profile_cells(const hs_rnn_desc* desc, const void* packed,
                         const void* x, const void* h0, const void* c0,
                         void* y, void* hn, void* cn,
                         void* workspace, size_t ws_bytes, void* stream,
                         float* cell_ms, float* forward_ms);

/* End-to-end forward on HOST buffers (the request path; pinned host memory
 * gives asynchronous copies).  x_host [T,B,I], h0_host/c0_host
 * [L*D,B,H] or NULL, outputs y_host [T,B,D*H], hn_host/cn_host [L*D,B,H].
 * x_dev/y_dev/hn_dev/cn_dev are caller-owned device staging buffers of the
 * same shapes; state_dev ([2][L*D,B,H], may be NULL without initial states)
 * stages h0/c0.  On the tensor-core path the copies overlap the compute: x is
 * uploaded in time chunks on an internal copy stream and each chunk's
 * layer-0 input projection starts when it lands; y is downloaded in time
 * chunks while the last layer's recurrence still runs (the copy stream
 * waits on per-step progress counters the kernel publishes).  All work,
 * copies included, is complete when `stream` reaches the end of the call.
 * Replaces: engine.simulate with io_transfers=True (engine.py:128-137,
 * 296-299, 375-378) — the host staging of entry inputs / exit outputs. */
int hs_rnn_forward_host(const hs_rnn_desc* desc, const void* packed,
                        const void* x_host, const void* h0_host, const void* c0_host,
                        void* y_host, void* hn_host, void* cn_host,
                        void* x_dev, void* y_dev, void* hn_dev, void* cn_dev, void* state_dev,
                        void* workspace, size_t ws_bytes, void* stream);

/* Completion of an async_outputs hs_rnn_forward_host call whose host output
 * buffer is `y_host` (the last such call on this thread and device): with
 * `stream` non-NULL, `stream` waits for its output copies; with NULL the
 * calling thread blocks until they are done.  A later forward that reuses
 * the same device staging buffers waits for them by itself. */
int hs_rnn_outputs_ready(const void* y_host, void* stream);

/* Convenience: pack + forward (weights in PyTorch layout).  Needs
 * packed_size + workspace bytes of workspace. */
int hs_rnn_forward(const hs_rnn_desc* desc, const void* x,
                   const void* const* w_ih, const void* const* w_hh,
                   const void* const* b_ih, const void* const* b_hh,
                   const void* h0, const void* c0, void* y, void* hn, void* cn,
                   void* workspace, size_t ws_bytes, void* stream);

/* Layer-pipeline stage link (the modelled link of
 * costmodel.py:133-139 / engine.py:317-339 made real).  A stage owns a range
 * of layers; its input arrives from the previous stage, its output goes to
 * the next, as bf16 hi/lo activation planes [2][T*B][I] (the layout the next
 * layer's input-projection GEMM reads) copied GPU-to-GPU by the copy engine
 * (NVLink P2P) in time chunks while the producing recurrence still runs.
 * All synchronisation is stream-ordered (cuStreamWaitValue32 /
 * cuStreamWriteValue32 on 32-bit words); no kernel spins on another GPU.
 * Counters are monotonic across requests, so they are never reset:
 *   x_avail   (consumer-owned) = x_base + timesteps of the current request
 *             present in x_planes; written by the producer after each chunk.
 *   consumed  (producer-owned) = set by the consumer to consumed_value once
 *             it has read its x_planes slot (its input GEMM is done with it).
 * Pointers to the peer's words / planes are mapped into this process by the
 * caller (CUDA IPC; paper_2307_11339_b200/parallel.py does it with
 * torch.multiprocessing's CUDA tensor sharing). */
typedef struct hs_stage_link {
  /* input side: NULL x_planes = the stage reads `x` (fp32) like a forward */
  const void* x_planes;           /* [2][T*B][I] bf16 hi/lo planes of this request's input */
  const uint32_t* x_avail;        /* local word the previous stage advances */
  uint32_t x_base;                /* value of *x_avail before this request's first chunk */
  uint32_t consumed_value;        /* written to *consumed_peer after the last read of x_planes */
  uint32_t* consumed_peer;        /* the previous stage's `consumed` word (peer memory) or NULL */
  /* output side: NULL y_peer_planes = no next stage (y is the model output) */
  void* y_peer_planes;            /* the next stage's x_planes slot for this request (peer memory) */
  uint32_t* y_peer_avail;         /* the next stage's x_avail word (peer memory) */
  uint32_t y_base;                /* *y_peer_avail before this request's first chunk */
  uint32_t consumed_wait;         /* wait until *consumed >= this before the first copy into the slot */
  const uint32_t* consumed;       /* local word the next stage advances (NULL = slot always free) */
  int32_t chunks;                 /* hand-off chunks per request (0 = 16) */
  int32_t reserved[5];
} hs_stage_link;

/* Sharing a stage's link buffers with the neighbouring stage's process (the
 * pipeline's setup step, SURVEY §8(b) "hs_pipeline_init"): export a device
 * pointer as a 64-byte CUDA IPC handle plus its offset inside the allocation,
 * import it in the other process (mapped once per allocation and process,
 * reference-counted), release the mapping when the pipeline is torn down.
 * Python callers can use torch.multiprocessing's CUDA sharing instead
 * (parallel.PeerPipeline does). */
int hs_pipeline_export(const void* dev_ptr, void* handle64, size_t* offset);
int hs_pipeline_import(const void* handle64, size_t offset, void** dev_ptr);
int hs_pipeline_release(void* dev_ptr);

/* One pipeline stage's forward (tensor-core path, unidirectional): as
 * hs_rnn_forward_packed over this stage's layers, with the input taken from
 * link->x_planes chunk by chunk as x_avail advances (the first layer's input
 * projection runs per arrived chunk), and the last layer's output shipped to
 * the next stage chunk by chunk as its recurrence publishes steps.  `y`
 * ([T, B, H] fp32) is written on every stage.  All work, copies and peer
 * signals included, is ordered on `stream`.  Replaces: the chunked
 * NCCL isend/irecv hand-off of parallel.LayerPipeline (round 1). */
int hs_rnn_forward_stage(const hs_rnn_desc* desc, const void* packed,
                         const void* x, const void* h0, const void* c0,
                         void* y, void* hn, void* cn, const hs_stage_link* link,
                         void* workspace, size_t ws_bytes, void* stream);

/* One GPU segment of a plan: timesteps t0..t1-1 (in the direction's own
 * processing order) of layer-direction `ld`.  On the tensor-core path the
 * segment runs the fused forward's kernels (split + K1 GEMM over the
 * segment's rows, then one recurrence launch of this layer-direction); shapes
 * the tensor-core path does not cover run the SIMT kernels.  `in` is that layer's input
 * [T, B, I_l], `out` its output [T, B, dirs*H] (columns d*H..d*H+H-1 are
 * written), `h_prev`/`c_prev` [B, H] the state entering step t0 and
 * `h_last`/`c_last` [B, H] receive the state after step t1-1.  `c_prev` and
 * `c_last` are ignored for GRU. */
int hs_rnn_run_cells(const hs_rnn_desc* desc, const void* packed, int32_t ld,
                     int32_t t0, int32_t t1, const void* in, void* out,
                     const void* h_prev, const void* c_prev,
                     void* h_last, void* c_last,
                     void* workspace, size_t ws_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HS_RNN_H */
