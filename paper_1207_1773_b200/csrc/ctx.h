// ctx.h — handle state of libeigb200 (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <set>
#include <string>
#include <utility>

#include "../../include/eig.h"
#include "kernels.h"

namespace eig {

enum WsId {
  WS_VXV = 0,     // s x 3nb: [V | X | V]
  WS_W,           // s x nb
  WS_PART,        // split-K partials
  WS_PART_SIDE,   // split-K partials of GEMMs on the side stream (concurrent with the main stream's)
  WS_SMALL,       // nb x nb scratch (Mh, M)
  WS_PANEL_REC,   // panel reduction records
  WS_BARRIER,     // grid barrier words
  WS_V,           // BT: explicit V_k
  WS_Y,           // BT: nb x m
  WS_Y2,          // BT: nb x m
  WS_TAGG,        // BT: aggregated T (ga*nb)^2 + Gram + temp
  WS_LINV,        // trsm: inverted diagonal blocks
  WS_T2,          // Q2 T factors
  WS_Q2PLAN,      // Q2 plan tables
  WS_Q2PROF,      // debug counters
  WS_Q2DONE,      // Q2 3M wavefront: per-block completion counters
  WS_BAND,        // hb2st band buffer (2nb+2 diagonals)
  WS_HBPROG,      // hb2st sweep progress flags
  WS_HBOFF,       // hb2st V2 slot offsets
  WS_HBMSG,       // hb2st position-stationary kernel: reflector / row messages
  WS_HBFLAG,      // ... and their flags
  WS_DC,          // stedc buffers
  WS_DC_SMALL,    // stedc per-level node tables
  WS_FRONT,       // potrf diagonal-block inverse
  WS_GST,         // hegst n x n scratch
  WS_INFO,        // device info word
  WS_SG_TAU1, WS_SG_T1, WS_SG_D, WS_SG_E, WS_SG_V2, WS_SG_TAU2, WS_SG_Z,   // solve_gen stage buffers
  WS_HOST_A, WS_HOST_V2, WS_HOST_TAU2, WS_HOST_L, WS_HOST_Z, WS_HOST_E, WS_HOST_TAU1, WS_HOST_T1,
  // collective calls (comm.cu): received factors on ranks > 0, packing, slices
  WS_C_A, WS_C_L, WS_C_PACK, WS_C_T1, WS_C_TAU1, WS_C_V2, WS_C_TAU2, WS_C_Z, WS_C_E, WS_C_STATUS,
  WS_C_ALOC, WS_C_DWORK,   // NEXT-4 distributed he2hb: this rank's columns, work
  WS_COUNT
};

struct Ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;        // high-priority stream for the he2hb panels (look-ahead)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t xfer = nullptr;        // host <-> device copies overlapped with compute (EIG_HOST_BUFFERS)
  cudaEvent_t ev_xfer = nullptr, ev_blk = nullptr;
  cudaEvent_t ev_q1[4] = {nullptr, nullptr, nullptr, nullptr};   // Q1: prep done [0,1], GEMMs done [2,3]
  int nb = 64;
  int q2g = 32;
  int num_sms = 148;
  int64_t launches = 0;
  // collective (multi-GPU) state: NCCL communicator and its stream (comm.cu)
  int rank = 0, nranks = 1;
  bool coll = false;
  void *nccl = nullptr;               // ncclComm_t
  cudaStream_t cstream = nullptr;     // NCCL collectives, pack / unpack
  cudaEvent_t ev_c[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t n_max = 0;
  unsigned flags = 0;
  bool use_3m = false;                // EIG_USE_3M: complex GEMMs as three real products
  // statistics of the last eig_hotpath / eig_solve_gen call (CUDA events)
  cudaEvent_t st_beg[EIG_NSTAGES] = {}, st_end[EIG_NSTAGES] = {};
  bool st_on[EIG_NSTAGES] = {};
  eig_stats st = {};
  void stat_reset() {
    for (int k = 0; k < EIG_NSTAGES; k++) st_on[k] = false;
    st = eig_stats();
    st.rank = rank;
    st.nranks = nranks;
  }
  int stat_begin(int k) { st_on[k] = true; return check(cudaEventRecord(st_beg[k], stream), "stat event"); }
  int stat_end(int k) { return check(cudaEventRecord(st_end[k], stream), "stat event"); }
  unsigned long long bar_epoch = 0;  // panel arrival counter value after the last launch
  unsigned long long *q2_prof = nullptr;  // debug: device counters for apply_q2 phases (EIG_Q2_PROFILE)
  std::string last_err;
  // Q2 plan tables (device, WS_Q2PLAN) for (q2_n, nb, q2g); q2_n = -1: none yet
  int64_t q2_n = -1;
  int q2_plan_nb = 0, q2_plan_g = 0;
  Q2Plan q2_plan;
  void *buf[WS_COUNT] = {};
  size_t bytes[WS_COUNT] = {};

  // Returns a device buffer of at least `need` bytes (grown, contents lost).
  void *ws(int id, size_t need);
  // Record a CUDA error; returns EIG_ERR_CUDA or 0.
  int check(cudaError_t e, const char *what);
  // Kernel attributes are per device: each handle (bound to one device, used
  // by one host thread) sets them once for its device before the first launch.
  std::set<std::pair<const void *, int>> attr_done;
  int func_attr(const void *f, cudaFuncAttribute attr, int value, const char *what) {
    const auto key = std::make_pair(f, (int)attr);
    if (attr_done.count(key)) return 0;
    const int rc = check(cudaFuncSetAttribute(f, attr, value), what);
    if (!rc) attr_done.insert(key);
    return rc;
  }
  int smem_attr(const void *f, int bytes, const char *what) {
    return func_attr(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes, what);
  }
  // After a kernel launch: count it and check for launch errors.
  int launched(const char *what) {
    launches++;
    return check(cudaGetLastError(), what);
  }
};

}  // namespace eig

#define EIG_TRY(x)            \
  do {                        \
    int _rc = (x);            \
    if (_rc) return _rc;      \
  } while (0)
