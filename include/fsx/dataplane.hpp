// fsx/dataplane.hpp -- one producer -> consumer data-plane pass in C++ over the
// C ABI: the native counterpart of paper_2603_12118_b200/dataplane.py.
//
// A pass is what the reference does per request between the encoder's
// emit_output (executor_sim.hpp:221-229, 321-336) and the LLM's admission
// (executor_sim.hpp:382-392), plus the merge the reference leaves out
// (SURVEY.md 8a-8):
//   alloc()    one receive-slab segment per item (fsx_slab_alloc_n: the
//              NodeArena policy, sidecar.hpp:149-163), all or nothing;
//   forward()  K1 pushes every item into its segment, chunk by chunk with a
//              completion flag per chunk (fsx_forward_batch);
//   merge()    K3 scans the placeholder rows and moves each item row into its
//              prompt row (fsx_merge), stream-ordered after forward() or with
//              early start on the chunk flags;
//   release()  the segments go back to the slab (the ack, sidecar.hpp:287-290).
// run_tee() is the N = 1 pass as ONE kernel (fsx_forward_merge): each item row
// is read once and stored into its slab segment (with the chunk flags) and
// into its prompt row.  run_place() is the slab-free alternative: the forward
// fused with the merge (fsx_forward_place), the producer's rows straight into
// the prompt rows.
// The batch's device arrays (prompt embedding, token ids, offsets, item
// views, scratch, status) are allocated once; a pass costs a handful of C-ABI
// calls and one small descriptor upload when segment offsets change.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsx.h"

namespace fsx {

class DataPlanePass {
 public:
  struct Item {
    const void* d_src;  // producer bytes on src_gpu's device (rows x row_bytes)
    int64_t rows;
  };
  struct Request {
    std::vector<int32_t> token_ids;  // prompt: text ids and placeholder_id rows
    std::vector<Item> items;         // input slots 1..m in items order
  };

  DataPlanePass(fsx_fabric* f, int src_gpu, int dst_gpu, int64_t row_bytes, int32_t placeholder_id,
                int64_t chunk_rows, const std::vector<Request>& reqs)
      : f_(f), src_(src_gpu), dst_(dst_gpu), rb_(row_bytes), pid_(placeholder_id), chunk_rows_(chunk_rows) {
    int dev = 0;
    check(fsx_device_of(f_, dst_gpu, &dev));
    dev_ = dev;
    std::vector<int64_t> req_row_off{0}, req_item_off{0}, item_row_off{0};
    std::vector<int32_t> tok;
    for (const Request& r : reqs) {
      tok.insert(tok.end(), r.token_ids.begin(), r.token_ids.end());
      req_row_off.push_back(req_row_off.back() + static_cast<int64_t>(r.token_ids.size()));
      for (const Item& it : r.items) {
        items_.push_back(it);
        item_row_off.push_back(item_row_off.back() + it.rows);
      }
      req_item_off.push_back(static_cast<int64_t>(items_.size()));
    }
    const int64_t R = static_cast<int64_t>(reqs.size()), M = static_cast<int64_t>(items_.size());
    total_rows_ = req_row_off.back();
    total_item_rows_ = item_row_off.back();
    cuda(cudaSetDevice(dev_));
    embeds_ = alloc_dev<uint8_t>(std::max<int64_t>(total_rows_ * rb_, 16));
    tok_ = upload(tok);
    req_row_off_ = upload(req_row_off);
    req_item_off_ = upload(req_item_off);
    item_row_off_ = upload(item_row_off);
    scratch_ = alloc_dev<int32_t>(std::max<int64_t>(total_item_rows_, 1));
    status_ = alloc_dev<int32_t>(std::max<int64_t>(R, 1));
    item_src_ = alloc_dev<const void*>(std::max<int64_t>(M, 1));
    xfers_.resize(static_cast<size_t>(M));
    lens_.resize(static_cast<size_t>(M));
    chunks_.resize(static_cast<size_t>(M));
    for (int64_t i = 0; i < M; ++i) {
      const int64_t nb = items_[i].rows * rb_, cb = chunk_rows_ > 0 ? chunk_rows_ * rb_ : 0;
      lens_[i] = nb;
      chunks_[i] = (cb <= 0 || cb >= nb) ? 1 : (nb + cb - 1) / cb;
      xfers_[i] = fsx_transfer{src_, dst_, items_[i].d_src, 0, nb, cb, 0, 0, nullptr};
      n_chunks_ += chunks_[i];
    }
    b_.num_requests = static_cast<int32_t>(R);
    b_.num_items = static_cast<int32_t>(M);
    b_.row_bytes = rb_;
    b_.placeholder_id = pid_;
    b_.mode = FSX_MERGE_FULL;
    b_.d_embeds = embeds_;
    b_.d_token_ids = tok_;
    b_.d_req_row_off = req_row_off_;
    b_.d_req_item_off = req_item_off_;
    b_.d_item_src = item_src_;
    b_.d_item_row_off = item_row_off_;
    b_.d_scratch = scratch_;
    b_.d_status = status_;
    b_.total_rows = total_rows_;
    b_.total_item_rows = total_item_rows_;
  }

  DataPlanePass(const DataPlanePass&) = delete;
  DataPlanePass& operator=(const DataPlanePass&) = delete;

  ~DataPlanePass() {
    if (held_) fsx_slab_free_n(f_, dst_, static_cast<int32_t>(offs_.size()), offs_.data());
    cudaSetDevice(dev_);
    cudaDeviceSynchronize();
    if (ev_ready_) {
      cudaEventDestroy(merged_ev_);
      for (auto& sl : stage_) {
        cudaFreeHost(sl.host);
        cudaEventDestroy(sl.ev);
      }
    }
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    for (void* p : owned_) cudaFree(p);
  }

  // Segments for every item; false (nothing held) when the slab is full.
  bool alloc() {
    offs_.assign(items_.size(), -1);
    check(fsx_slab_alloc_n(f_, dst_, static_cast<int32_t>(items_.size()), lens_.data(), offs_.data()));
    if (!items_.empty() && offs_[0] < 0) return false;
    held_ = true;
    if (offs_ != uploaded_offs_) {  // first fit hands back the same offsets pass after pass
      void* base = nullptr;
      check(fsx_slab_ptr(f_, dst_, 0, &base));
      std::vector<const void*> views(items_.size());
      for (size_t i = 0; i < items_.size(); ++i) views[i] = static_cast<const uint8_t*>(base) + offs_[i];
      cuda(cudaSetDevice(dev_));
      if (!views.empty())
        cuda(cudaMemcpy(item_src_, views.data(), views.size() * sizeof(void*), cudaMemcpyHostToDevice));
      uploaded_offs_ = offs_;
    }
    return true;
  }

  // K1 for every item (flags drawn from the consumer slab's ring).
  void forward(cudaStream_t st, uint32_t options = 0) {
    if (items_.empty()) return;
    int64_t fb = 0;
    check(fsx_flags_alloc(f_, dst_, static_cast<int32_t>(n_chunks_), &fb));
    for (size_t i = 0; i < items_.size(); ++i) {
      xfers_[i].dst_off = offs_[i];
      xfers_[i].flag_base = fb;
      xfers_[i].token = 0;
      fb += chunks_[i];
    }
    check(fsx_forward_batch(f_, static_cast<int32_t>(items_.size()), xfers_.data(), options, st));
  }

  // K3, stream-ordered after forward() on the same stream.
  void merge(cudaStream_t st) { check(fsx_merge(f_, dst_, &b_, st)); }

  void release() {
    if (!held_) return;
    check(fsx_slab_free_n(f_, dst_, static_cast<int32_t>(offs_.size()), offs_.data()));
    held_ = false;
  }

  // alloc -> forward -> merge -> release; false when the slab was full.
  bool run(cudaStream_t st, uint32_t fwd_options = 0) {
    if (!alloc()) return false;
    forward(st, fwd_options);
    merge(st);
    release();  // host bookkeeping; the next pass's K1 is stream-ordered after this merge
    return true;
  }

  // The colocated pass (producer and consumer on the same GPU): K1 on
  // `k1_stream`, the early-start merge on `merge_stream` (create it with the
  // highest priority) following K1 chunk by chunk, one CTA per SM, merged
  // slab rows discarded from L2 (FSX_MERGE_COLOCATED | FSX_MERGE_DISCARD;
  // DESIGN.md §3).  The next pass's K1 waits for this pass's merge (slab
  // reuse).  False when the slab was full.
  bool run_colocated(cudaStream_t k1_stream, cudaStream_t merge_stream) {
    if (!alloc()) return false;
    if (!ev_ready_) {
      cuda(cudaSetDevice(dev_));
      cuda(cudaEventCreateWithFlags(&merged_ev_, cudaEventDisableTiming));
      for (auto& sl : stage_) {
        cuda(cudaHostAlloc(&sl.host, 2 * std::max<size_t>(items_.size(), 1) * sizeof(uint64_t),
                           cudaHostAllocDefault));
        sl.dev = alloc_dev<uint64_t>(2 * std::max<int64_t>(static_cast<int64_t>(items_.size()), 1));
        cuda(cudaEventCreateWithFlags(&sl.ev, cudaEventDisableTiming));
      }
      std::vector<int64_t> cr(items_.size());
      for (size_t i = 0; i < items_.size(); ++i) cr[i] = chunk_rows_ > 0 ? chunk_rows_ : items_[i].rows;
      chunk_rows_dev_ = upload(cr);
      uint64_t* f0 = nullptr;
      check(fsx_flag_ptr(f_, dst_, 0, &f0));
      flag0_ = f0;
      ev_ready_ = true;
    } else {
      cuda(cudaStreamWaitEvent(k1_stream, merged_ev_, 0));  // pass s-1 merged: segments free
    }
    forward(k1_stream);
    // early-start descriptors: (flag pointer, token) per item, staged in a
    // pinned ring slot whose previous upload has run
    Stage& sl = stage_[next_stage_];
    next_stage_ = (next_stage_ + 1) % kStages;
    cuda(cudaEventSynchronize(sl.ev));
    const size_t M = items_.size();
    for (size_t i = 0; i < M; ++i) {
      sl.host[i] = reinterpret_cast<uint64_t>(flag0_ + xfers_[i].flag_base);
      sl.host[M + i] = xfers_[i].token;
    }
    cuda(cudaMemcpyAsync(sl.dev, sl.host, 2 * M * sizeof(uint64_t), cudaMemcpyHostToDevice, merge_stream));
    cuda(cudaEventRecord(sl.ev, merge_stream));
    fsx_merge_batch mb = b_;
    mb.mode = FSX_MERGE_FULL | FSX_MERGE_COLOCATED | FSX_MERGE_DISCARD;
    mb.d_item_flag = reinterpret_cast<const uint64_t* const*>(sl.dev);
    mb.d_item_token = sl.dev + M;
    mb.d_item_chunk_rows = chunk_rows_dev_;
    check(fsx_merge(f_, dst_, &mb, merge_stream));
    cuda(cudaEventRecord(merged_ev_, merge_stream));
    release();
    return true;
  }

  // The tee pass (producer and consumer on the same device): alloc, then one
  // fsx_forward_merge (scan + the fused forward/merge kernel, stream order),
  // then release.  Same slab segments and chunk flags as run(), same merged
  // rows, the payload crossing HBM three times instead of four.
  bool run_tee(cudaStream_t st, uint32_t fwd_options = 0) {
    if (!alloc()) return false;
    ensure_place_src();
    int64_t fb = 0;
    if (!items_.empty()) check(fsx_flags_alloc(f_, dst_, static_cast<int32_t>(n_chunks_), &fb));
    for (size_t i = 0; i < items_.size(); ++i) {
      xfers_[i].dst_off = offs_[i];
      xfers_[i].flag_base = fb;
      xfers_[i].token = 0;
      fb += chunks_[i];
    }
    fsx_merge_batch mb = b_;
    mb.d_item_src = place_src_;
    check(fsx_forward_merge(f_, static_cast<int32_t>(items_.size()), xfers_.data(), &mb, fwd_options, st));
    release();
    return true;
  }

  // Direct placement (fsx_forward_place): the forward fused with the merge.
  // The producer writes every item row from its own buffer straight into the
  // consumer's placeholder rows (scan + row copy, one fsx call, stream order);
  // no slab segment is held and the payload crosses memory once.  Always
  // succeeds (nothing to allocate).
  bool run_place(cudaStream_t st) {
    ensure_place_src();
    fsx_merge_batch mb = b_;
    mb.d_item_src = place_src_;
    check(fsx_forward_place(f_, src_, dst_, &mb, -1, 0, st));
    return true;
  }

  // CUDA-graph form of the stream-ordered pass for launch-bound batches:
  // capture() records forward + merge once (segment offsets, flag ranges and
  // tokens are baked in: the same first-fit offsets come back every pass, and
  // nothing waits on the flags in stream order); run_graph() then does the
  // host bookkeeping (alloc, release) and one graph launch per pass.
  void capture(cudaStream_t st) {
    if (!alloc()) throw std::runtime_error("fsx: slab full while capturing the pass");
    cuda(cudaSetDevice(dev_));
    cuda(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    forward(st);
    merge(st);
    cudaGraph_t g = nullptr;
    cuda(cudaStreamEndCapture(st, &g));
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    cuda(cudaGraphInstantiate(&graph_exec_, g, 0));
    cudaGraphDestroy(g);
    captured_offs_ = offs_;
    release();
  }

  bool run_graph(cudaStream_t st) {
    if (!graph_exec_) throw std::runtime_error("fsx: capture() the pass first");
    if (!alloc()) return false;
    if (offs_ != captured_offs_) {  // the slab moved under us: re-record
      release();
      capture(st);
      if (!alloc()) return false;
    }
    cuda(cudaGraphLaunch(graph_exec_, st));
    release();
    return true;
  }

  uint8_t* embeds() const { return embeds_; }
  const int32_t* status() const { return status_; }
  int64_t total_rows() const { return total_rows_; }
  int64_t total_item_rows() const { return total_item_rows_; }
  int64_t payload_bytes() const { return total_item_rows_ * rb_; }
  int device() const { return dev_; }

 private:
  static void check(int rc) {
    if (rc != FSX_OK) throw std::runtime_error(std::string("fsx: ") + fsx_last_error());
  }
  static void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("cuda: ") + cudaGetErrorString(e));
  }
  // Device array of the producer's item pointers (tee and direct placement).
  void ensure_place_src() {
    if (place_src_) return;
    std::vector<const void*> src(items_.size());
    for (size_t i = 0; i < items_.size(); ++i) src[i] = items_[i].d_src;
    cuda(cudaSetDevice(dev_));
    place_src_ = upload(src);
  }
  template <class T>
  T* alloc_dev(int64_t n) {
    void* p = nullptr;
    cuda(cudaMalloc(&p, static_cast<size_t>(n) * sizeof(T)));
    owned_.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const std::vector<T>& v) {
    T* p = alloc_dev<T>(std::max<int64_t>(static_cast<int64_t>(v.size()), 1));
    if (!v.empty()) cuda(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  }

  fsx_fabric* f_;
  int src_, dst_, dev_ = 0;
  int64_t rb_;
  int32_t pid_;
  int64_t chunk_rows_;
  std::vector<Item> items_;
  int64_t total_rows_ = 0, total_item_rows_ = 0, n_chunks_ = 0;
  std::vector<fsx_transfer> xfers_;
  std::vector<int64_t> lens_, chunks_, offs_, uploaded_offs_;
  bool held_ = false;
  std::vector<void*> owned_;
  uint8_t* embeds_ = nullptr;
  int32_t* tok_ = nullptr;
  int64_t *req_row_off_ = nullptr, *req_item_off_ = nullptr, *item_row_off_ = nullptr;
  int32_t *scratch_ = nullptr, *status_ = nullptr;
  const void** item_src_ = nullptr;
  const void** place_src_ = nullptr;  // producer buffers, for run_tee / run_place
  fsx_merge_batch b_{};
  // colocated pass state
  static constexpr int kStages = 4;
  struct Stage {
    uint64_t* host = nullptr;
    uint64_t* dev = nullptr;
    cudaEvent_t ev = nullptr;
  };
  Stage stage_[kStages];
  int next_stage_ = 0;
  bool ev_ready_ = false;
  cudaEvent_t merged_ev_ = nullptr;
  int64_t* chunk_rows_dev_ = nullptr;
  uint64_t* flag0_ = nullptr;
  // graph form
  cudaGraphExec_t graph_exec_ = nullptr;
  std::vector<int64_t> captured_offs_;
};

}  // namespace fsx
