// Device-resident verification engine behind the C ABI (spin_ctx).
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <map>
#include <mutex>
#include <thread>
#include <string>
#include <memory>
#include <tuple>
#include <vector>

#include "gemm.cuh"
#include "kernels.cuh"
#include "spin_c.h"

namespace spin {

// One model (target or SSM): synthetic bf16 weights, KV cache, RoPE tables.
struct ModelDev {
  spin_model_desc d{};
  int D = 0, H = 0, hd = 0, F = 0, V = 0, L = 0;
  bf16* wbuf = nullptr;
  bf16* sbuf = nullptr;  // draft-path slab copies of the layer weights (SSMs)
  bf16* emb = nullptr;
  bf16* head = nullptr;
  std::vector<LayerW> layers;
  bf16* kc = nullptr;
  bf16* vc = nullptr;
  float* rcos = nullptr;
  float* rsin = nullptr;
  CUtensorMap tm_k{}, tm_v{};
  size_t weight_bytes = 0, kv_bytes = 0;
};

// Forward workspace of one model (one stream at a time).
struct Lane {
  int T_cap = 0, R_cap = 0, seg_cap = 0, rows_cap = 0, piece_cap = 0;
  FwdMeta meta{};
  float* h = nullptr;
  bf16 *xn = nullptr, *attn = nullptr, *act = nullptr;
  float* q = nullptr;
  float* ssp = nullptr;  // draft path: per-unit sums of squares of h [T][D / 16]
  bf16* hb = nullptr;    // draft path: bf16 copy of h [T][D]
  float* part = nullptr;
  AttnWork aw{};
  float* amax_val = nullptr;
  int32_t* amax_idx = nullptr;
  float* logits = nullptr;
  int head_sms = 0;  // SMs the lm_head GEMM may use (0 = all): off the critical chain, fewer
  std::vector<void*> allocs;
};

// Kernel classes of profile_round (spin_c.h SPIN_PROF_*).
enum ProfCat : int {
  kProfTargetGemm = 0,
  kProfTargetHead = 1,
  kProfTargetAttn = 2,
  kProfTargetEpi = 3,
  kProfSsmGemm = 4,
  kProfSsmHead = 5,
  kProfSsmAttn = 6,
  kProfSsmEpi = 7,
  kProfMeta = 8,
  kProfCats = 9,
};

struct FwdShape {
  int T, R, rows, qmax;
  // 1: every request's new KV rows are exactly its query positions (verify, draft
  // steps), so attention may fetch older keys before the projection completes; 0 for
  // extends, whose virtual requests read keys written earlier in the same forward.
  int early = 0;
};

class Engine {
 public:
  Engine(const spin_model_desc& target, const spin_model_desc* ssms, int n_ssm, const spin_engine_opts& opts);
  ~Engine();

  void prefill(int n, const int32_t* slots, const int32_t* lens, const int32_t* prompts);
  // prewarm (optional, [n]): destination SSM to warm for request i while this round runs
  void round(int n, const int32_t* slots, const int32_t* ssm_of, const int32_t* prewarm, spin_round_out* out);
  void run_rounds(int n, const int32_t* slots, const int32_t* ssm_of, int rounds, int64_t* emitted, float* ms);
  // synchronous KV catch-up (switches); positions recomputed, per request in per_req
  int64_t switch_ssm(int n, const int32_t* slots, const int32_t* ssm_of, int32_t* per_req = nullptr);
  void read_tokens(int slot, int32_t* tokens, int cap, int32_t* len);
  void read_logits(float* logits, int64_t cap, int32_t* rows);
  // One round without graphs, with CUDA events around every launch; per
  // kernel class: device ms, algorithmic bytes (GEMMs), launches.
  void profile_round(int n, const int32_t* slots, const int32_t* ssm_of, double* ms, double* bytes,
                     int64_t* launches);
  int64_t launches_per_round(int n, const int32_t* slots, const int32_t* ssm_of);
  // Per-SSM draft end of the last round, ms after the round start (-1: SSM idle).
  void last_round_trace(float* spec_end_ms, int cap) const;
  void kernel_bench(int kind, int iters, double* us_per_launch, double* bytes_per_launch);
  void verify_bench(int n, const int32_t* slots, const int32_t* draft_lens, const int32_t* drafts, int packed,
                    int iters, spin_verify_stats* out);

 private:
  struct RoundPlan;
  // Speculation/verification pipelining (simulate_pipelined,
  // pipeline.cpp:160-329): each SSM's requests split into micro-batch groups; a unit
  // (SSM j, group g) drafts on j's stream and is verified on its own, FIFO on sv_; the
  // next slot's draft of a unit starts as soon as that unit was verified (causality,
  // pipeline.cpp:236-241), so drafting overlaps the verification of other units.
  struct PipeUnit {
    int ssm = 0, g = 0, n = 0;
    int off_list = 0, off_ssm_of = 0, off_out = 0;
    double arrival = 0.0;  // expected draft end (verify FIFO order)
    cudaGraph_t gd = nullptr, gv = nullptr;
    cudaGraphExec_t draft = nullptr, verify = nullptr;
    cudaEvent_t ev_d = nullptr, ev_v = nullptr;             // ordering
    cudaEvent_t t_d = nullptr, t_v0 = nullptr, t_v1 = nullptr;  // timing
  };
  struct PipePlan {
    std::vector<PipeUnit> units;  // SSM-major, groups in order (draft order per stream)
    std::vector<int> vorder;      // verify order (expected arrival)
    int in_ints = 0, out_ints = 0, n_act = 0;
    int64_t launches = 0;
  };
  std::vector<int> mb_;  // micro-batches per SSM; all ones = the serial round
  std::map<std::vector<int>, std::unique_ptr<PipePlan>> pipes_;
  bool pipelined() const {
    for (int b : mb_)
      if (b != 1) return true;
    return false;
  }
  PipePlan& plan_pipe(int n, const int32_t* ssm_of);
  void stage_pipe(PipePlan& pp, int n, const int32_t* slots, const int32_t* ssm_of);
  void launch_pipe_slot(PipePlan& pp, bool first, bool host_round);

 public:
  void set_micro_batches(const int32_t* per_ssm, int m);
  void get_micro_batches(int32_t* per_ssm, int m) const;
  void tune_micro_batches(int n, const int32_t* slots, const int32_t* ssm_of, int max_mb, int probe_rounds,
                          double threshold, int32_t* chosen, double* curve, int curve_cap, int* n_curve);

 private:
  void init_model(ModelDev& m, const spin_model_desc& d, bool draft);
  void init_lane(Lane& ln, const ModelDev& m, int T_cap, int R_cap, bool logits);
  void forward(ModelDev& m, Lane& ln, const FwdShape& sh, cudaStream_t s, int head_mode);
  void forward_draft(ModelDev& m, Lane& ln, const FwdShape& sh, AttnGeom g, cudaStream_t s, int head_mode);
  bool draft_fused_ = true;
  // SPIN_STAMPS=<csv path>: per-CTA globaltimer stamps of the draft kernels, dumped after
  // every round (launch, kind, cta, start, after-wait, after-main-loop, end) -- a
  // profiling aid for latency-bound kernel chains.
  unsigned long long* stamps_ = nullptr;
  size_t stamp_cap_ = 0, stamp_used_ = 0;
  std::vector<std::array<int, 3>> stamp_tab_;  // kind, ctas, offset
  std::string stamp_path_;
  unsigned long long* stamp_slot(int kind, int ctas);
  void dump_stamps();
  void extend(int model, const std::vector<std::tuple<int, int, int>>& ranges, cudaStream_t s = nullptr,
              Lane* lane = nullptr, int32_t* pinned = nullptr, size_t pinned_cap = 0);  // (slot, from, to)
  void join_prewarm();
  void enqueue_prewarm(int n, const int32_t* slots, const int32_t* prewarm, const int32_t* ssm_of);
  void init_prewarm();
  // prewarm: per SSM a lane, a stream, staging and a completion event
  std::vector<Lane> pwlane_;
  std::vector<cudaStream_t> ps_;
  std::vector<cudaEvent_t> ev_pw_;
  // staging (row metadata, ssm_len values) in two halves per SSM, alternating per job, so a
  // job never waits for the previous one's catch-up to finish before it can stage
  std::vector<int32_t*> pw_pin_;  // [2 * M]
  std::vector<cudaEvent_t> ev_pw_stage_;  // [2 * M]: the job that staged in half b is done
  std::vector<int> pw_half_;
  size_t pw_pin_cap_ = 0;
  std::vector<char> pw_pending_;
  std::thread pw_thread_;  // enqueues the prewarm extends while the round runs
  std::vector<int32_t*> pw_len_pin_;  // [2 * M] pinned ssm_len values the prewarm stream uploads
  bool pw_error_ = false;
  std::string pw_error_msg_;
  int64_t pw_tokens_ = 0;
  float last_switch_ms_ = 0.f;
  cudaEvent_t ev_r0_ = nullptr, ev_r1_ = nullptr;
  RoundPlan& plan_round(int n, const int32_t* slots, const int32_t* ssm_of);
  void capture_round(RoundPlan& p);
  void enqueue_draft(int j, const int32_t* d_list, int nj, cudaStream_t sj);
  void enqueue_verify(const int32_t* d_list, const int32_t* d_ssm_of, int n, int32_t* d_out, cudaStream_t s);
  void record_timing(cudaEvent_t ev, cudaStream_t s);
  void prof_begin(int cat, cudaStream_t s);
  void prof_end(cudaStream_t s, double bytes);
  bool capturing_ = false;
  bool prof_ = false;
  std::atomic<int64_t> launches_{0};
  std::mutex plan_mu_;  // plans_ is shared with the prewarm thread
  struct ProfRec {
    int cat;
    cudaEvent_t a, b;
    double bytes;
  };
  std::vector<ProfRec> prof_recs_;
  void sync_state_from_device();
  void sync_sv(const char* what);  // synchronise sv_ and raise a flagged device status
  volatile int32_t* h_err_ = nullptr;
  int32_t* d_err_ = nullptr;

  spin_engine_opts opts_{};
  int num_sms_ = 148;
  ModelDev target_;
  std::vector<ModelDev> ssm_;
  Lane tlane_;
  std::vector<Lane> slane_;
  SlotState st_{};
  cudaStream_t sv_ = nullptr;
  std::vector<cudaStream_t> ss_;
  std::map<std::tuple<int, int, int, int, int>, GemmPlan> plans_;
  const GemmPlan& plan(int n_out, int k, int t, int mode, int sms = 0);  // sms: SMs the plan may use (0 = all)
  std::vector<void*> plan_tables_;

  // host mirror of the per-slot state
  std::vector<int32_t> h_tokens_, h_committed_, h_ssm_len_;
  bool mirror_stale_ = false;

  // round staging (pinned) + device copies
  int32_t* pin_in_ = nullptr;   // lists
  int32_t* pin_out_ = nullptr;  // outcomes
  int32_t* d_in_ = nullptr;
  int32_t* d_out_ = nullptr;
  unsigned long long* d_emitted_ = nullptr;
  size_t in_cap_ = 0, out_cap_ = 0;
  cudaEvent_t ev_fork_ = nullptr, ev_start_ = nullptr, ev_draft_ = nullptr, ev_end_ = nullptr;
  std::vector<cudaEvent_t> ev_join_, ev_spec_end_;
  std::vector<float> last_spec_ms_;
  std::map<std::vector<int>, std::unique_ptr<RoundPlan>> rounds_;
  int last_verify_rows_ = 0;
};

}  // namespace spin
