// Multi-GPU slab domain decomposition behind the C-ABI (include/pmg_b200.h,
// pmg_dd_*): the smoother, V-cycle and full multigrid of
// /root/reference/proj/src/multigrid.cpp:313-400 (smoother.cpp:41-151 per
// level) on `world` ranks, one device each, in C++ over CUDA streams / events
// and either device copies (cudaMemcpyPeerAsync over NVLink, or plain D2D for
// virtual ranks sharing a GPU) or NCCL point-to-point / collectives.
//
// Decomposition (the same plan as paper_2405_19004_b200/dd.py,
// which runs it over torch.distributed and is tested against the numpy
// oracle on CPU):
//   * rank g owns the patch-vertex planes v_z in [a_g, b_g] of the level; it
//     keeps the global dof planes E = [lo - H, hi + H] (H = 4k + 4 halo) where
//     [lo, hi] = [k(a-1)-1, k(b+1)-1] is what its patches read;
//   * smoother, per colour: the boundary-layer patches (v = a or b) on a side
//     stream, then ONE one-directional k-plane message per interface (which
//     side sends is fixed by the colour's z-parity, patches.cpp:31-33), the
//     interior patches concurrently on the main stream;
//   * V-cycle: halo(x) -> r = b - Ax on owned planes -> halo(r) -> b_c = R r
//     on coarse owned planes -> halo(b_c) -> recurse -> halo(x_c) ->
//     x += P x_c on [lo, hi] -> post-smooth. Levels on which a rank would own
//     fewer than 2H planes are agglomerated on rank 0: the coarse owned shares
//     of R r are gathered there, rank 0 runs the rest of the V-cycle as one
//     CUDA graph of its single-device context and broadcasts x_c.
// Every value is computed by the single-device kernels' per-output arithmetic
// (the *_slab entry points of capi.cu), so P ranks reproduce one device
// bitwise; only the norms (rank-ordered sums of per-rank partial sums) round
// differently.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <set>
#include <vector>

#include "blas.cuh"
#include "capi_internal.hpp"

using namespace pmgb;

namespace
{

struct InvalidArg : std::invalid_argument
{
  using std::invalid_argument::invalid_argument;
};

// a status of an inner C-ABI call becomes the matching exception again
void ck(int status, const char *what)
{
  if (status == PMG_OK)
    return;
  const std::string msg = std::string(what) + ": " + pmg_last_error();
  if (status == PMG_ERR_INVALID)
    throw InvalidArg(msg);
  if (status == PMG_ERR_CUDA)
    throw CudaError(msg);
  throw std::runtime_error(msg);
}

// ---------------------------------------------------------------------------
// NCCL, loaded on first use (the library itself does not link it)
// ---------------------------------------------------------------------------
struct Nccl
{
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl &nccl()
{
  static std::once_flag once;
  static Nccl n;
  static std::string err;
  std::call_once(once, [] {
    // the copy torch already loaded (same soname) when it is in the process
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h)
    {
      err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char *name) {
      void *p = dlsym(h, name);
      if (!p && err.empty())
        err = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommInitAll = reinterpret_cast<decltype(n.CommInitAll)>(sym("ncclCommInitAll"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
    n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
    n.Broadcast = reinterpret_cast<decltype(n.Broadcast)>(sym("ncclBroadcast"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
  });
  if (!err.empty())
    throw std::runtime_error(err);
  return n;
}

void ckn(ncclResult_t r, const char *what)
{
  if (r != ncclSuccess)
    throw std::runtime_error(std::string(what) + ": " + nccl().GetErrorString(r));
}

// ---------------------------------------------------------------------------
// The plan (dd.py make_plan / colour_step / level_slab / decomposed_levels)
// ---------------------------------------------------------------------------
struct Plan
{
  int world = 1, rank = 0, k = 1, n = 2, nz = 2;
  int a = 1, b = 1;          // owned vertex planes (1-based lattice vertex index)
  int64_t lo = 0, hi = 0;    // dof planes the rank's patches read (inclusive)
  int64_t own_lo = 0, own_hi = 0;
  int64_t m = 1, mz = 1;
};

Plan make_plan(int world, int rank, int k, int level, int stack)
{
  Plan p;
  p.world = world;
  p.rank = rank;
  p.k = k;
  p.n = 1 << level;
  p.nz = stack * p.n;
  const int nv = p.nz - 1;
  if (nv < world)
    throw InvalidArg(std::to_string(nv) + " vertex planes cannot be split over " + std::to_string(world) +
                     " ranks");
  p.a = 1 + static_cast<int>((static_cast<int64_t>(rank) * nv) / world);
  p.b = static_cast<int>((static_cast<int64_t>(rank + 1) * nv) / world);
  p.m = static_cast<int64_t>(p.n) * k - 1;
  p.mz = static_cast<int64_t>(p.nz) * k - 1;
  p.lo = std::max<int64_t>(0, static_cast<int64_t>(k) * (p.a - 1) - 1);
  p.hi = std::min<int64_t>(p.mz - 1, static_cast<int64_t>(k) * (p.b + 1) - 1);
  p.own_lo = rank == 0 ? 0 : static_cast<int64_t>(k) * (p.a - 1);
  p.own_hi = rank == world - 1 ? p.mz - 1 : static_cast<int64_t>(k) * p.b - 1;
  return p;
}

bool colour_nonempty(int n, int color)
{
  for (int a = 0; a < 2; ++a)
    if (((color >> a) & 1 ? n / 2 : n / 2 - 1) <= 0)
      return false;
  return true;
}

struct Msg
{
  int peer;
  int64_t g0, np;  // global first plane, planes
};

struct ColourStep
{
  std::vector<std::pair<int, int>> early, late;  // vertex-plane ranges
  std::vector<Msg> sends, recvs;
};

ColourStep colour_step(const Plan &p, int color)
{
  ColourStep st;
  if (!colour_nonempty(p.n, color))
    return st;
  const int zb = (color >> 2) & 1, k = p.k;
  std::set<int> early;
  if (p.rank + 1 < p.world)  // upper interface
  {
    if (p.b % 2 == zb)
    {
      st.sends.push_back({p.rank + 1, static_cast<int64_t>(k) * p.b - 1, k});
      early.insert(p.b);
    }
    else
      st.recvs.push_back({p.rank + 1, static_cast<int64_t>(k) * p.b, k});
  }
  if (p.rank > 0)  // lower interface (the neighbour's b is a - 1)
  {
    const int bl = p.a - 1;
    if (bl % 2 == zb)
      st.recvs.push_back({p.rank - 1, static_cast<int64_t>(k) * bl - 1, k});
    else
    {
      st.sends.push_back({p.rank - 1, static_cast<int64_t>(k) * bl, k});
      early.insert(p.a);
    }
  }
  for (int v : early)
    st.early.push_back({v, v});
  const int lo_v = p.a + (early.count(p.a) ? 1 : 0);
  const int hi_v = p.b - ((early.count(p.b) && p.b != p.a) ? 1 : 0);
  if (lo_v <= hi_v)
    st.late.push_back({lo_v, hi_v});
  return st;
}

int halo_width(int k) { return 4 * k + 4; }

struct Slab
{
  Plan plan;
  int64_t e0 = 0, e1 = 0;  // planes held (inclusive)
  int64_t np() const { return e1 - e0 + 1; }
};

Slab level_slab(int world, int rank, int k, int level, int stack)
{
  Slab s;
  s.plan = make_plan(world, rank, k, level, stack);
  const int H = halo_width(k);
  s.e0 = std::max<int64_t>(0, s.plan.lo - H);
  s.e1 = std::min<int64_t>(s.plan.mz - 1, s.plan.hi + H);
  return s;
}

// levels (finest first) on which every rank owns >= 2H dof planes
std::vector<int> decomposed_levels(int world, int k, int finest)
{
  std::vector<int> out;
  for (int lev = finest; lev >= 2; --lev)
  {
    if ((1 << lev) - 1 < world)
      break;
    int64_t thinnest = INT64_MAX;
    for (int r = 0; r < world; ++r)
    {
      const Plan p = make_plan(world, r, k, lev, 1);
      thinnest = std::min(thinnest, p.own_hi - p.own_lo + 1);
    }
    if (thinnest < 2 * halo_width(k))
      break;
    out.push_back(lev);
  }
  return out;
}

// planes of my E owned by a neighbour (recvs) and of the neighbour's E owned
// by me (sends), in global planes (dd.py _exchange_specs)
void exchange_specs(const std::vector<Slab> &all, int rank, std::vector<Msg> &sends, std::vector<Msg> &recvs)
{
  const Slab &me = all[rank];
  for (int q : {rank - 1, rank + 1})
  {
    if (q < 0 || q >= static_cast<int>(all.size()))
      continue;
    const Slab &nb = all[q];
    int64_t lo = std::max(me.e0, nb.plan.own_lo), hi = std::min(me.e1, nb.plan.own_hi);
    if (lo <= hi)
      recvs.push_back({q, lo, hi - lo + 1});
    lo = std::max(nb.e0, me.plan.own_lo);
    hi = std::min(nb.e1, me.plan.own_hi);
    if (lo <= hi)
      sends.push_back({q, lo, hi - lo + 1});
  }
}

// ---------------------------------------------------------------------------
// per-rank state
// ---------------------------------------------------------------------------
enum Arr
{
  A_X = 0,  // x of the level (finest: owned; coarser decomposed: the finer level's A_XC)
  A_B,      // b of the level (finest: owned; coarser: the finer level's A_BC)
  A_R,      // residual (owned planes valid after residual + halo)
  A_XC,     // x of the level below: its slab (E planes), or the whole agglomerated level
  A_BC,     // b of the level below, same shape
  A_NUM
};

struct LevelState
{
  bool active = false;
  Slab slab;
  pmg_level lv = nullptr;         // this level's setup on the rank's device
  char *a[A_NUM] = {};            // the level's arrays (views)
  DevBuf own[A_NUM];              // storage of the arrays this level owns
  std::vector<Msg> hsend, hrecv;  // halo exchange (decomposed levels and the finest)
  ColourStep steps[8];
};

struct Rank
{
  int rank = 0, device = 0;
  cudaStream_t main = nullptr, side = nullptr;
  cudaEvent_t ev_start = nullptr, ev_early = nullptr, ev_side = nullptr, ev_pt = nullptr, ev_pulled = nullptr;
  std::unique_ptr<LevelState[]> L;  // indexed by mesh level (0 unused)
  int nlev = 0;
  pmg_level agg_lv = nullptr; // setup of the agglomerated partner level (restrict / prolongate slabs)
  DevBuf red;                 // reduction partials + result
  ncclComm_t comm = nullptr;
  pmg_mg root_mg = nullptr;     // rank 0: the agglomerated levels as one single-device context
  DevBuf fmg_x[32], fmg_b[32];  // rank 0: nested-iteration vectors of the agglomerated levels
};

}  // namespace

struct pmg_dd_s
{
  int world = 1, dim = 3, k = 1, finest = 1, stack = 1, dtype = PMG_F64, variant = PMG_FUSED;
  int transport = PMG_DD_COPY;
  int pre = 1, post = 1;
  size_t ts = 8;
  std::vector<int> dd_levels;  // decomposed levels, finest first (empty: the V-cycle runs on rank 0)
  int agg = 0;                 // finest agglomerated mesh level
  std::vector<std::unique_ptr<Rank>> local;
  bool use_graph = false;                 // pmg_dd_set_graph: smoothing step / V-cycle as CUDA graphs
  bool capturing = false;                 // inside a capture: the coarse V-cycle runs eagerly (captured)
  cudaGraphExec_t smooth_graph = nullptr, vcycle_graph = nullptr;
  cudaEvent_t fork = nullptr;
  std::vector<cudaEvent_t> joins;

  ~pmg_dd_s()
  {
    if (!local.empty())
    {
      cudaSetDevice(local[0]->device);
      if (smooth_graph)
        cudaGraphExecDestroy(smooth_graph);
      if (vcycle_graph)
        cudaGraphExecDestroy(vcycle_graph);
      if (fork)
        cudaEventDestroy(fork);
      for (cudaEvent_t e : joins)
        cudaEventDestroy(e);
    }
    for (auto &r : local)
    {
      cudaSetDevice(r->device);
      cudaDeviceSynchronize();
      for (int l = 0; l < r->nlev; ++l)
      {
        LevelState &ls = r->L[l];
        if (ls.lv)
          pmg_level_destroy(ls.lv);
        for (auto &b : ls.own)
          b.~DevBuf(), new (&b) DevBuf();
      }
      if (r->agg_lv)
        pmg_level_destroy(r->agg_lv);
      if (r->root_mg)
        pmg_mg_destroy(r->root_mg);
      for (cudaEvent_t e : {r->ev_start, r->ev_early, r->ev_side, r->ev_pt, r->ev_pulled})
        if (e)
          cudaEventDestroy(e);
      if (r->main)
        cudaStreamDestroy(r->main);
      if (r->side)
        cudaStreamDestroy(r->side);
      if (r->comm)
        nccl().CommDestroy(r->comm);
      r->red.~DevBuf(), new (&r->red) DevBuf();
      for (auto &b : r->fmg_x)
        b.~DevBuf(), new (&b) DevBuf();
      for (auto &b : r->fmg_b)
        b.~DevBuf(), new (&b) DevBuf();
    }
  }

  bool nccl_mode() const { return transport == PMG_DD_NCCL; }
  Rank *find(int rank) const
  {
    for (auto &r : local)
      if (r->rank == rank)
        return r.get();
    return nullptr;
  }
  int64_t m(int lev) const { return static_cast<int64_t>(1 << lev) * k - 1; }
  int64_t ps(int lev) const { return m(lev) * m(lev); }
  int64_t mz(int lev) const { return static_cast<int64_t>(stack) * (1 << lev) * k - 1; }
  bool is_dd(int lev) const { return std::find(dd_levels.begin(), dd_levels.end(), lev) != dd_levels.end(); }
  size_t bytes(int64_t words) const { return static_cast<size_t>(words) * ts; }
  pmg_level lv(Rank &r, int lev) const { return r.L[lev].active ? r.L[lev].lv : r.agg_lv; }
};

namespace
{

template <typename F>
int dd_guard(F &&f)
{
  return capi_guard(std::forward<F>(f));
}

// planes [g0, g0 + np) of two arrays that hold global planes from e0 on
void copy_planes(pmg_dd_s *d, Rank &dst, char *dst_base, int64_t dst_e0, Rank &src, const char *src_base,
                 int64_t src_e0, int64_t g0, int64_t np, int64_t ps, cudaStream_t s)
{
  const size_t bytes = d->bytes(np * ps);
  if (bytes == 0)
    return;
  char *to = dst_base + d->bytes((g0 - dst_e0) * ps);
  const char *from = src_base + d->bytes((g0 - src_e0) * ps);
  if (dst.device == src.device)
    check_cuda(cudaMemcpyAsync(to, from, bytes, cudaMemcpyDeviceToDevice, s), "D2D plane copy");
  else
    check_cuda(cudaMemcpyPeerAsync(to, dst.device, from, src.device, bytes, s), "peer plane copy");
}

// grouped NCCL point-to-point of plane ranges of one array per local rank
void nccl_p2p(pmg_dd_s *d, int lev, bool side, const std::vector<const std::vector<Msg> *> &sends,
              const std::vector<const std::vector<Msg> *> &recvs, const std::vector<char *> &base,
              const std::vector<int64_t> &e0, int64_t ps)
{
  const Nccl &N = nccl();
  (void)lev;
  ckn(N.GroupStart(), "ncclGroupStart");
  for (size_t i = 0; i < d->local.size(); ++i)
  {
    Rank &r = *d->local[i];
    cudaStream_t s = side ? r.side : r.main;
    for (const Msg &m : *sends[i])
      ckn(N.Send(base[i] + d->bytes((m.g0 - e0[i]) * ps), d->bytes(m.np * ps), ncclChar, m.peer, r.comm, s),
          "ncclSend");
    for (const Msg &m : *recvs[i])
      ckn(N.Recv(base[i] + d->bytes((m.g0 - e0[i]) * ps), d->bytes(m.np * ps), ncclChar, m.peer, r.comm, s),
          "ncclRecv");
  }
  ckn(N.GroupEnd(), "ncclGroupEnd");
}

// ---- halo exchange of array `arr` of level lev (main streams) --------------
void halo(pmg_dd_s *d, int lev, int arr)
{
  const int64_t ps = d->ps(lev);
  if (d->nccl_mode())
  {
    std::vector<const std::vector<Msg> *> s, r;
    std::vector<char *> base;
    std::vector<int64_t> e0;
    for (auto &rp : d->local)
    {
      s.push_back(&rp->L[lev].hsend);
      r.push_back(&rp->L[lev].hrecv);
      base.push_back(rp->L[lev].a[arr]);
      e0.push_back(rp->L[lev].slab.e0);
    }
    nccl_p2p(d, lev, false, s, r, base, e0, ps);
    return;
  }
  // copies: the receiver pulls after the owner's point, the owner waits for
  // the pulls before it touches the planes again
  for (auto &rp : d->local)
  {
    DevScope g(rp->device);
    check_cuda(cudaEventRecord(rp->ev_pt, rp->main), "event");
  }
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    DevScope g(r.device);
    LevelState &ls = r.L[lev];
    for (const Msg &m : ls.hrecv)
    {
      Rank &q = *d->find(m.peer);
      check_cuda(cudaStreamWaitEvent(r.main, q.ev_pt, 0), "wait");
      copy_planes(d, r, ls.a[arr], ls.slab.e0, q, q.L[lev].a[arr], q.L[lev].slab.e0, m.g0, m.np, ps, r.main);
    }
    check_cuda(cudaEventRecord(r.ev_pulled, r.main), "event");
  }
  for (auto &rp : d->local)
  {
    DevScope g(rp->device);
    for (const Msg &m : rp->L[lev].hsend)
      check_cuda(cudaStreamWaitEvent(rp->main, d->find(m.peer)->ev_pulled, 0), "wait");
  }
}

// ---- one smoothing step of level lev (smoother.cpp:41-151 on the slabs) ----
void smooth_level(pmg_dd_s *d, int lev)
{
  const int64_t ps = d->ps(lev);
  for (int c = 0; c < 8; ++c)
  {
    for (auto &rp : d->local)
    {
      Rank &r = *rp;
      DevScope g(r.device);
      check_cuda(cudaEventRecord(r.ev_start, r.main), "event");
      check_cuda(cudaStreamWaitEvent(r.side, r.ev_start, 0), "wait");
      LevelState &ls = r.L[lev];
      for (auto [v0, v1] : ls.steps[c].early)
        ck(pmg_smooth_color_slab(ls.lv, d->variant, c, ls.a[A_X], ls.a[A_B], ls.slab.e0, ls.slab.plan.nz, v0, v1,
                                 r.side),
           "dd smooth (boundary layer)");
      check_cuda(cudaEventRecord(r.ev_early, r.side), "event");
    }
    if (d->nccl_mode())
    {
      std::vector<const std::vector<Msg> *> s, rv;
      std::vector<char *> base;
      std::vector<int64_t> e0;
      for (auto &rp : d->local)
      {
        s.push_back(&rp->L[lev].steps[c].sends);
        rv.push_back(&rp->L[lev].steps[c].recvs);
        base.push_back(rp->L[lev].a[A_X]);
        e0.push_back(rp->L[lev].slab.e0);
      }
      nccl_p2p(d, lev, true, s, rv, base, e0, ps);
    }
    else
    {
      for (auto &rp : d->local)
      {
        Rank &r = *rp;
        DevScope g(r.device);
        LevelState &ls = r.L[lev];
        for (const Msg &m : ls.steps[c].recvs)
        {
          Rank &q = *d->find(m.peer);
          check_cuda(cudaStreamWaitEvent(r.side, q.ev_early, 0), "wait");
          copy_planes(d, r, ls.a[A_X], ls.slab.e0, q, q.L[lev].a[A_X], q.L[lev].slab.e0, m.g0, m.np, ps, r.side);
        }
      }
    }
    for (auto &rp : d->local)
    {
      Rank &r = *rp;
      DevScope g(r.device);
      check_cuda(cudaEventRecord(r.ev_side, r.side), "event");
      LevelState &ls = r.L[lev];
      for (auto [v0, v1] : ls.steps[c].late)
        ck(pmg_smooth_color_slab(ls.lv, d->variant, c, ls.a[A_X], ls.a[A_B], ls.slab.e0, ls.slab.plan.nz, v0, v1,
                                 r.main),
           "dd smooth (interior)");
    }
    for (auto &rp : d->local)
    {
      Rank &r = *rp;
      DevScope g(r.device);
      check_cuda(cudaStreamWaitEvent(r.main, r.ev_side, 0), "wait");
      if (!d->nccl_mode())  // the ranks that pulled from me are done with my planes
        for (const Msg &m : r.L[lev].steps[c].sends)
          check_cuda(cudaStreamWaitEvent(r.main, d->find(m.peer)->ev_side, 0), "wait");
    }
  }
}

// ---- agglomeration on rank 0 -------------------------------------------------
// every rank holds its planes [share[r].first, share[r].second) of a whole
// vector in `arr` of level lev (np planes of ps words): collect them on rank 0
void gather_to_root(pmg_dd_s *d, int lev, int arr, const std::vector<std::pair<int64_t, int64_t>> &share, int64_t ps)
{
  if (d->nccl_mode())
  {
    std::vector<std::vector<Msg>> s(d->local.size()), r(d->local.size());
    std::vector<const std::vector<Msg> *> sp, rp_;
    std::vector<char *> base;
    std::vector<int64_t> e0;
    for (size_t i = 0; i < d->local.size(); ++i)
    {
      Rank &rk = *d->local[i];
      if (rk.rank == 0)
      {
        for (int q = 1; q < d->world; ++q)
          r[i].push_back({q, share[q].first, share[q].second - share[q].first});
      }
      else
        s[i].push_back({0, share[rk.rank].first, share[rk.rank].second - share[rk.rank].first});
      sp.push_back(&s[i]);
      rp_.push_back(&r[i]);
      base.push_back(rk.L[lev].a[arr]);
      e0.push_back(0);
    }
    nccl_p2p(d, lev, false, sp, rp_, base, e0, ps);
    return;
  }
  Rank &root = *d->find(0);
  for (auto &rp : d->local)
  {
    DevScope g(rp->device);
    check_cuda(cudaEventRecord(rp->ev_pt, rp->main), "event");
  }
  {
    DevScope g(root.device);
    for (auto &rp : d->local)
    {
      if (rp->rank == 0)
        continue;
      const auto [q0, q1] = share[rp->rank];
      check_cuda(cudaStreamWaitEvent(root.main, rp->ev_pt, 0), "wait");
      copy_planes(d, root, root.L[lev].a[arr], 0, *rp, rp->L[lev].a[arr], 0, q0, q1 - q0, ps, root.main);
    }
    check_cuda(cudaEventRecord(root.ev_pulled, root.main), "event");
  }
  for (auto &rp : d->local)
    if (rp->rank != 0)
    {
      DevScope g(rp->device);
      check_cuda(cudaStreamWaitEvent(rp->main, root.ev_pulled, 0), "wait");
    }
}

// `words` values of rank 0's `arr` (level lev) to every rank
void broadcast_from_root(pmg_dd_s *d, int lev, int arr, int64_t words)
{
  if (d->nccl_mode())
  {
    const Nccl &N = nccl();
    ckn(N.GroupStart(), "ncclGroupStart");
    for (auto &rp : d->local)
    {
      char *base = rp->L[lev].a[arr];
      ckn(N.Broadcast(base, base, d->bytes(words), ncclChar, 0, rp->comm, rp->main), "ncclBroadcast");
    }
    ckn(N.GroupEnd(), "ncclGroupEnd");
    return;
  }
  Rank &root = *d->find(0);
  {
    DevScope g(root.device);
    check_cuda(cudaEventRecord(root.ev_pt, root.main), "event");
  }
  for (auto &rp : d->local)
  {
    if (rp->rank == 0)
      continue;
    DevScope g(rp->device);
    check_cuda(cudaStreamWaitEvent(rp->main, root.ev_pt, 0), "wait");
    copy_planes(d, *rp, rp->L[lev].a[arr], 0, root, root.L[lev].a[arr], 0, 0, words, 1, rp->main);
    check_cuda(cudaEventRecord(rp->ev_pulled, rp->main), "event");
  }
  DevScope g(root.device);
  for (auto &rp : d->local)
    if (rp->rank != 0)
      check_cuda(cudaStreamWaitEvent(root.main, rp->ev_pulled, 0), "wait");
}

// coarse planes [q0, q1) of level lev-1 a rank restricts at the agglomeration
// boundary: a partition of [0, mc) proportional to the fine ownership
std::vector<std::pair<int64_t, int64_t>> coarse_shares(const pmg_dd_s *d, int lev)
{
  std::vector<std::pair<int64_t, int64_t>> share(d->world);
  const int64_t mc = d->m(lev - 1);
  for (int q = 0; q < d->world; ++q)
  {
    const Plan p = make_plan(d->world, q, d->k, lev, 1);
    share[q].first = q == 0 ? 0 : (p.own_lo * mc) / p.mz;
    share[q].second = q == d->world - 1 ? mc : ((p.own_hi + 1) * mc) / p.mz;
  }
  return share;
}

// ---- the V-cycle of decomposed level lev (multigrid.cpp:313-348) -----------
void vcycle_level(pmg_dd_s *d, int lev)
{
  for (int i = 0; i < d->pre; ++i)
    smooth_level(d, lev);
  halo(d, lev, A_X);
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    LevelState &ls = r.L[lev];
    const Plan &p = ls.slab.plan;
    ck(pmg_compute_residual_slab(ls.lv, ls.a[A_X], ls.a[A_B], ls.a[A_R], ls.slab.e0, ls.slab.np(), p.own_lo,
                                 p.own_hi + 1, r.main),
       "dd residual");
  }
  halo(d, lev, A_R);
  const int cl = lev - 1;
  if (d->is_dd(cl))
  {
    for (auto &rp : d->local)
    {
      Rank &r = *rp;
      LevelState &ls = r.L[lev], &lc = r.L[cl];
      const Plan &pc = lc.slab.plan;
      ck(pmg_restrict_slab(lc.lv, ls.lv, ls.a[A_R], ls.slab.e0, ls.slab.np(), ls.a[A_BC], lc.slab.e0, lc.slab.np(),
                           pc.own_lo, pc.own_hi + 1, r.main),
         "dd restrict");
    }
    halo(d, cl, A_B);  // the coarse level's b is this level's b_c
    for (auto &rp : d->local)
    {
      DevScope g(rp->device);
      check_cuda(cudaMemsetAsync(rp->L[lev].a[A_XC], 0, d->bytes(rp->L[cl].slab.np() * d->ps(cl)), rp->main),
                 "x_c = 0");
    }
    vcycle_level(d, cl);
    halo(d, cl, A_X);
  }
  else
  {
    // agglomerated coarse level: shares of R r -> rank 0, V-cycle there, x_c back
    const auto share = coarse_shares(d, lev);
    for (auto &rp : d->local)
    {
      Rank &r = *rp;
      LevelState &ls = r.L[lev];
      const auto [q0, q1] = share[r.rank];
      ck(pmg_restrict_slab(d->lv(r, cl), ls.lv, ls.a[A_R], ls.slab.e0, ls.slab.np(), ls.a[A_BC], 0, d->mz(cl), q0,
                           q1, r.main),
         "dd restrict (agglomeration)");
    }
    gather_to_root(d, lev, A_BC, share, d->ps(cl));
    if (Rank *root = d->find(0))
    {
      DevScope g(root->device);
      // the recursion starts from x_c = 0 (multigrid.cpp:336)
      check_cuda(cudaMemsetAsync(root->L[lev].a[A_XC], 0, d->bytes(d->mz(cl) * d->ps(cl)), root->main), "x_c = 0");
      // as the single-device recursion does it (multigrid.cpp:335-338)
      mg_coarse_correction(root->root_mg, cl - 1, root->L[lev].a[A_XC], root->L[lev].a[A_BC], !d->capturing,
                           root->main);
    }
    broadcast_from_root(d, lev, A_XC, d->mz(cl) * d->ps(cl));
  }
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    LevelState &ls = r.L[lev];
    int64_t e0c = 0, npc = d->mz(cl);
    if (d->is_dd(cl))
    {
      e0c = r.L[cl].slab.e0;
      npc = r.L[cl].slab.np();
    }
    ck(pmg_prolongate_slab(d->lv(r, cl), ls.lv, ls.a[A_XC], e0c, npc, ls.a[A_X], ls.slab.e0, ls.slab.np(),
                           ls.slab.plan.lo, ls.slab.plan.hi + 1, 1, r.main),
       "dd prolongate");
  }
  for (int i = 0; i < d->post; ++i)
    smooth_level(d, lev);
}

// ---- finest level too thin to split: the whole V-cycle on rank 0 -----------
void vcycle_agglomerated(pmg_dd_s *d)
{
  const int lev = d->finest;
  const int64_t ps = d->ps(lev);
  std::vector<std::pair<int64_t, int64_t>> share(d->world);
  for (int q = 0; q < d->world; ++q)
  {
    const Plan p = make_plan(d->world, q, d->k, lev, 1);
    share[q] = {p.own_lo, p.own_hi + 1};
  }
  // owned planes of x and b into the whole-level buffers
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    DevScope g(r.device);
    LevelState &ls = r.L[lev];
    const auto [o0, o1] = share[r.rank];
    copy_planes(d, r, ls.a[A_XC], 0, r, ls.a[A_X], ls.slab.e0, o0, o1 - o0, ps, r.main);
    copy_planes(d, r, ls.a[A_BC], 0, r, ls.a[A_B], ls.slab.e0, o0, o1 - o0, ps, r.main);
  }
  gather_to_root(d, lev, A_XC, share, ps);
  gather_to_root(d, lev, A_BC, share, ps);
  if (Rank *root = d->find(0))
  {
    DevScope g(root->device);
    ck(pmg_v_cycle(root->root_mg, lev - 1, root->L[lev].a[A_XC], root->L[lev].a[A_BC], d->capturing ? 0 : 1,
                   root->main),
       "dd V-cycle (agglomerated)");
  }
  broadcast_from_root(d, lev, A_XC, d->mz(lev) * ps);
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    DevScope g(r.device);
    LevelState &ls = r.L[lev];
    copy_planes(d, r, ls.a[A_X], ls.slab.e0, r, ls.a[A_XC], 0, ls.slab.e0, ls.slab.np(), ps, r.main);
  }
}

void vcycle_finest(pmg_dd_s *d)
{
  if (d->dd_levels.empty())
    vcycle_agglomerated(d);
  else
    vcycle_level(d, d->finest);
}

// all-reduced Euclidean norm of the owned planes of `arr` of the finest level
// (vector_norm, multigrid.cpp:260-266; partial sums added in rank order)
double norm_owned(pmg_dd_s *d, int arr)
{
  const int lev = d->finest;
  const int64_t ps = d->ps(lev);
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    DevScope g(r.device);
    LevelState &ls = r.L[lev];
    const Plan &p = ls.slab.plan;
    const char *v = ls.a[arr] + d->bytes((p.own_lo - ls.slab.e0) * ps);
    const int64_t n = (p.own_hi - p.own_lo + 1) * ps;
    double *red = r.red.as<double>();
    if (d->dtype == PMG_F64)
      launch_dot<double>(reinterpret_cast<const double *>(v), reinterpret_cast<const double *>(v), n, red,
                         red + RED_BLOCKS, false, r.main);
    else
      launch_dot<float>(reinterpret_cast<const float *>(v), reinterpret_cast<const float *>(v), n, red,
                        red + RED_BLOCKS, false, r.main);
  }
  if (d->nccl_mode())
  {
    const Nccl &N = nccl();
    ckn(N.GroupStart(), "ncclGroupStart");
    for (auto &rp : d->local)
    {
      double *res = rp->red.as<double>() + RED_BLOCKS;
      ckn(N.AllReduce(res, res, 1, ncclFloat64, ncclSum, rp->comm, rp->main), "ncclAllReduce");
    }
    ckn(N.GroupEnd(), "ncclGroupEnd");
    Rank &r = *d->local[0];
    DevScope g(r.device);
    double out = 0;
    check_cuda(cudaMemcpyAsync(&out, r.red.as<double>() + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, r.main),
               "D2H");
    check_cuda(cudaStreamSynchronize(r.main), "sync");
    return std::sqrt(out);
  }
  double sum = 0.0;
  for (auto &rp : d->local)  // rank order
  {
    Rank &r = *rp;
    DevScope g(r.device);
    double part = 0;
    check_cuda(cudaMemcpyAsync(&part, r.red.as<double>() + RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, r.main),
               "D2H");
    check_cuda(cudaStreamSynchronize(r.main), "sync");
    sum += part;
  }
  return std::sqrt(sum);
}

// r = b - A x on the owned planes of the finest level
void residual_finest(pmg_dd_s *d)
{
  const int lev = d->finest;
  halo(d, lev, A_X);
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    LevelState &ls = r.L[lev];
    const Plan &p = ls.slab.plan;
    ck(pmg_compute_residual_slab(ls.lv, ls.a[A_X], ls.a[A_B], ls.a[A_R], ls.slab.e0, ls.slab.np(), p.own_lo,
                                 p.own_hi + 1, r.main),
       "dd residual");
  }
}

// host global vector of level lev -> the slabs (E planes) of array arr
void scatter_host(pmg_dd_s *d, int lev, int arr, const void *global)
{
  const int64_t ps = d->ps(lev);
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    DevScope g(r.device);
    LevelState &ls = r.L[lev];
    check_cuda(cudaMemcpyAsync(ls.a[arr], static_cast<const char *>(global) + d->bytes(ls.slab.e0 * ps),
                               d->bytes(ls.slab.np() * ps), cudaMemcpyHostToDevice, r.main),
               "scatter H2D");
    check_cuda(cudaStreamSynchronize(r.main), "sync");
  }
}

void sync_all(pmg_dd_s *d)
{
  for (auto &rp : d->local)
  {
    DevScope g(rp->device);
    check_cuda(cudaStreamSynchronize(rp->main), "dd synchronize");
    check_cuda(cudaStreamSynchronize(rp->side), "dd synchronize");
  }
}

void build(pmg_dd_s *d, const std::vector<std::pair<int, int>> &ranks_devices)
{
  if (d->dim != 3)
    throw InvalidArg("dd: the slab decomposition is 3D (dim must be 3)");
  if (d->stack < 1)
    throw InvalidArg("dd: stack must be >= 1");
  if (d->k < 1 || d->k > 7 || d->finest < 1)
    throw InvalidArg("dd: degree must be 1..7 and finest_level >= 1");
  if (d->variant != PMG_FUSED && d->variant != PMG_BOUNDARY)
    throw InvalidArg("dd: the slab smoother supports the fused and boundary variants");
  if (d->dtype != PMG_F64 && d->dtype != PMG_F32)
    throw InvalidArg("dtype must be PMG_F64 or PMG_F32");
  d->ts = d->dtype == PMG_F64 ? 8 : 4;
  (void)make_plan(d->world, 0, d->k, d->finest, d->stack);  // validates the split
  if (d->stack == 1)
    d->dd_levels = decomposed_levels(d->world, d->k, d->finest);
  if (!d->dd_levels.empty() && d->dd_levels.front() != d->finest)
    d->dd_levels.clear();
  d->agg = d->dd_levels.empty() ? d->finest : d->dd_levels.back() - 1;
  const int F = d->finest;
  for (auto [rank, dev] : ranks_devices)
  {
    auto r = std::make_unique<Rank>();
    r->rank = rank;
    r->device = dev;
    DevScope g(dev);
    check_cuda(cudaStreamCreateWithFlags(&r->main, cudaStreamNonBlocking), "stream");
    check_cuda(cudaStreamCreateWithFlags(&r->side, cudaStreamNonBlocking), "stream");
    for (cudaEvent_t *e : {&r->ev_start, &r->ev_early, &r->ev_side, &r->ev_pt, &r->ev_pulled})
      check_cuda(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "event");
    r->red.ensure((RED_BLOCKS + 8) * sizeof(double));
    r->L.reset(new LevelState[F + 1]);
    r->nlev = F + 1;
    std::vector<int> levs = d->dd_levels;
    if (levs.empty())
      levs.push_back(F);
    for (int lev : levs)
    {
      LevelState &ls = r->L[lev];
      ls.active = true;
      ls.slab = level_slab(d->world, rank, d->k, lev, lev == F ? d->stack : 1);
      ck(pmg_level_create(3, d->k, lev, d->dtype, dev, &ls.lv), "dd level");
      for (int c = 0; c < 8; ++c)
        ls.steps[c] = colour_step(ls.slab.plan, c);
    }
    if (!d->dd_levels.empty() && d->agg >= 1)
      ck(pmg_level_create(3, d->k, d->agg, d->dtype, dev, &r->agg_lv), "dd level");
    if (rank == 0 && d->stack == 1)
    {
      ck(pmg_mg_create(3, d->k, d->agg, d->dtype, d->variant, dev, &r->root_mg), "dd coarse context");
      ck(pmg_mg_set_smoothing(r->root_mg, d->pre, d->post), "dd coarse context");
    }
    d->local.push_back(std::move(r));
  }
  // halo specs (decomposed levels; the finest always, for the residual)
  std::vector<int> hl = d->dd_levels;
  if (hl.empty() && d->stack == 1)
    hl.push_back(F);
  for (int lev : hl)
  {
    std::vector<Slab> all;
    for (int q = 0; q < d->world; ++q)
      all.push_back(level_slab(d->world, q, d->k, lev, 1));
    for (auto &rp : d->local)
      exchange_specs(all, rp->rank, rp->L[lev].hsend, rp->L[lev].hrecv);
  }
  // arrays
  for (auto &rp : d->local)
  {
    Rank &r = *rp;
    DevScope g(r.device);
    auto alloc = [&](LevelState &ls, int arr, int64_t words) {
      ls.own[arr].ensure(d->bytes(words) + 16);
      check_cuda(cudaMemset(ls.own[arr].p, 0, ls.own[arr].bytes), "memset");
      ls.a[arr] = ls.own[arr].as<char>();
    };
    LevelState &lf = r.L[F];
    const int64_t fw = lf.slab.np() * d->ps(F);
    alloc(lf, A_X, fw);
    alloc(lf, A_B, fw);
    if (d->stack != 1)
      continue;
    alloc(lf, A_R, fw);
    if (d->dd_levels.empty())
    {
      alloc(lf, A_XC, d->mz(F) * d->ps(F));  // whole-level gather buffers
      alloc(lf, A_BC, d->mz(F) * d->ps(F));
      continue;
    }
    for (int lev : d->dd_levels)
    {
      LevelState &ls = r.L[lev];
      if (lev != F)
      {
        ls.a[A_X] = r.L[lev + 1].a[A_XC];  // the recursion's x_c / b_c
        ls.a[A_B] = r.L[lev + 1].a[A_BC];
        alloc(ls, A_R, ls.slab.np() * d->ps(lev));
      }
      const int cl = lev - 1;
      const int64_t cw = d->is_dd(cl) ? r.L[cl].slab.np() * d->ps(cl) : d->mz(cl) * d->ps(cl);
      alloc(ls, A_XC, cw);
      alloc(ls, A_BC, cw);
    }
  }
}

void check_vcycle(const pmg_dd_s *d, const char *what)
{
  if (d->stack != 1)
    throw InvalidArg(std::string(what) + ": the V-cycle is defined on the unit cube (stack = 1)");
}

}  // namespace

// one eager V-cycle with the finest x saved and restored: allocations of the
// coarse single-device context (first use of its levels) happen outside a
// capture
static void vcycle_warm(pmg_dd_s *d)
{
  std::vector<DevBuf> save(d->local.size());
  for (size_t i = 0; i < d->local.size(); ++i)
  {
    Rank &r = *d->local[i];
    DevScope g(r.device);
    LevelState &ls = r.L[d->finest];
    const size_t bytes = d->bytes(ls.slab.np() * d->ps(d->finest));
    save[i].ensure(bytes);
    check_cuda(cudaMemcpyAsync(save[i].p, ls.a[A_X], bytes, cudaMemcpyDeviceToDevice, r.main), "save x");
  }
  vcycle_finest(d);
  for (size_t i = 0; i < d->local.size(); ++i)
  {
    Rank &r = *d->local[i];
    DevScope g(r.device);
    LevelState &ls = r.L[d->finest];
    check_cuda(cudaMemcpyAsync(ls.a[A_X], save[i].p, save[i].bytes, cudaMemcpyDeviceToDevice, r.main), "restore x");
  }
  sync_all(d);
}

static bool dd_graphable(const pmg_dd_s *d)
{
  for (auto &r : d->local)
    if (r->device != d->local[0]->device)
      return false;
  return true;
}

template <typename F>
static void dd_capture(pmg_dd_s *d, cudaGraphExec_t &exec, F &&body)
{
  Rank &r0 = *d->local[0];
  DevScope g(r0.device);
  if (!d->fork)
    check_cuda(cudaEventCreateWithFlags(&d->fork, cudaEventDisableTiming), "event");
  while (d->joins.size() < d->local.size())
  {
    cudaEvent_t e;
    check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    d->joins.push_back(e);
  }
  sync_all(d);
  cudaGraph_t graph = nullptr;
  check_cuda(cudaStreamBeginCapture(r0.main, cudaStreamCaptureModeRelaxed), "capture begin");
  try
  {
    check_cuda(cudaEventRecord(d->fork, r0.main), "event");
    for (size_t i = 1; i < d->local.size(); ++i)
      check_cuda(cudaStreamWaitEvent(d->local[i]->main, d->fork, 0), "wait");
    d->capturing = true;
    body();
    d->capturing = false;
    for (size_t i = 1; i < d->local.size(); ++i)
    {
      check_cuda(cudaEventRecord(d->joins[i], d->local[i]->main), "event");
      check_cuda(cudaStreamWaitEvent(r0.main, d->joins[i], 0), "wait");
    }
  }
  catch (...)
  {
    d->capturing = false;
    cudaStreamEndCapture(r0.main, &graph);
    if (graph)
      cudaGraphDestroy(graph);
    throw;
  }
  check_cuda(cudaStreamEndCapture(r0.main, &graph), "capture end");
  check_cuda(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
}

extern "C" {

// host-only view of the decomposition plan (tests compare it with dd.py):
// out[0..6] = a, b, lo, hi, own_lo, own_hi, decomposed (this level is split
// with a 2H halo); then per colour c: n_early, n_sends, n_recvs followed by
// the early vertex planes and (peer, g0, np) per send / recv; returns the
// number of int64 written (or PMG_ERR_INVALID via a negative count).
int64_t pmg_dd_plan(int world, int rank, int degree, int level, int stack, int64_t *out, int64_t cap)
{
  int64_t n = -1;
  const int st = dd_guard([&] {
    if (!out || world < 1 || rank < 0 || rank >= world || degree < 1 || level < 1 || stack < 1)
      throw InvalidArg("dd_plan: invalid arguments");
    const Plan p = make_plan(world, rank, degree, level, stack);
    std::vector<int64_t> v = {p.a, p.b, p.lo, p.hi, p.own_lo, p.own_hi};
    const auto dl = stack == 1 ? decomposed_levels(world, degree, level) : std::vector<int>{};
    v.push_back(std::find(dl.begin(), dl.end(), level) != dl.end() ? 1 : 0);
    for (int c = 0; c < 8; ++c)
    {
      const ColourStep cs = colour_step(p, c);
      v.push_back(static_cast<int64_t>(cs.early.size()));
      v.push_back(static_cast<int64_t>(cs.sends.size()));
      v.push_back(static_cast<int64_t>(cs.recvs.size()));
      for (auto [lo, hi] : cs.early)
        v.push_back(lo);
      for (const auto *lst : {&cs.sends, &cs.recvs})
        for (const Msg &m : *lst)
        {
          v.push_back(m.peer);
          v.push_back(m.g0);
          v.push_back(m.np);
        }
    }
    if (static_cast<int64_t>(v.size()) > cap)
      throw InvalidArg("dd_plan: output capacity too small");
    std::copy(v.begin(), v.end(), out);
    n = static_cast<int64_t>(v.size());
  });
  return st == PMG_OK ? n : -static_cast<int64_t>(st);
}

int pmg_dd_nccl_id(void *id_out)
{
  return dd_guard([&] {
    if (!id_out)
      throw InvalidArg("null id");
    ncclUniqueId id;
    ckn(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int pmg_dd_create(int ndev, const int *devices, int dim, int degree, int finest_level, int stack, int dtype,
                  int variant, int transport, pmg_dd *out)
{
  return dd_guard([&] {
    if (!out || !devices || ndev < 1)
      throw InvalidArg("dd_create: invalid arguments");
    if (transport != PMG_DD_COPY && transport != PMG_DD_NCCL)
      throw InvalidArg("dd_create: unknown transport");
    int count = 0;
    check_cuda(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    std::vector<std::pair<int, int>> rd;
    for (int i = 0; i < ndev; ++i)
    {
      if (devices[i] < 0 || devices[i] >= count)
        throw InvalidArg("dd_create: no such CUDA device " + std::to_string(devices[i]));
      rd.push_back({i, devices[i]});
    }
    if (transport == PMG_DD_NCCL && static_cast<int>(std::set<int>(devices, devices + ndev).size()) != ndev)
      throw InvalidArg("dd_create: NCCL needs one distinct device per rank (PMG_DD_COPY runs virtual ranks)");
    auto d = std::make_unique<pmg_dd_s>();
    d->world = ndev;
    d->dim = dim;
    d->k = degree;
    d->finest = finest_level;
    d->stack = stack;
    d->dtype = dtype;
    d->variant = variant;
    d->transport = transport;
    build(d.get(), rd);
    // direct peer copies (NVLink copy engines) between distinct devices
    for (int i = 0; i < ndev; ++i)
      for (int j = 0; j < ndev; ++j)
        if (devices[i] != devices[j])
        {
          int ok = 0;
          check_cuda(cudaDeviceCanAccessPeer(&ok, devices[i], devices[j]), "cudaDeviceCanAccessPeer");
          if (!ok)
            continue;
          DevScope g(devices[i]);
          const cudaError_t e = cudaDeviceEnablePeerAccess(devices[j], 0);
          if (e == cudaErrorPeerAccessAlreadyEnabled)
            cudaGetLastError();
          else
            check_cuda(e, "cudaDeviceEnablePeerAccess");
        }
    if (transport == PMG_DD_NCCL)
    {
      std::vector<ncclComm_t> comms(ndev);
      ckn(nccl().CommInitAll(comms.data(), ndev, devices), "ncclCommInitAll");
      for (int i = 0; i < ndev; ++i)
        d->local[i]->comm = comms[i];
    }
    *out = d.release();
  });
}

int pmg_dd_create_rank(int world, int rank, int device, const void *nccl_id, int dim, int degree, int finest_level,
                       int stack, int dtype, int variant, pmg_dd *out)
{
  return dd_guard([&] {
    if (!out || !nccl_id || world < 1 || rank < 0 || rank >= world)
      throw InvalidArg("dd_create_rank: invalid arguments");
    int count = 0;
    check_cuda(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (device < 0 || device >= count)
      throw InvalidArg("dd_create_rank: no such CUDA device " + std::to_string(device));
    auto d = std::make_unique<pmg_dd_s>();
    d->world = world;
    d->dim = dim;
    d->k = degree;
    d->finest = finest_level;
    d->stack = stack;
    d->dtype = dtype;
    d->variant = variant;
    d->transport = PMG_DD_NCCL;
    build(d.get(), {{rank, device}});
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    DevScope g(device);
    ckn(nccl().CommInitRank(&d->local[0]->comm, world, id, rank), "ncclCommInitRank");
    *out = d.release();
  });
}

int pmg_dd_destroy(pmg_dd h)
{
  return dd_guard([&] { delete h; });
}

int pmg_dd_info(pmg_dd h, int *world, int *local_ranks, int *decomposed)
{
  return dd_guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    if (world)
      *world = h->world;
    if (local_ranks)
      *local_ranks = static_cast<int>(h->local.size());
    if (decomposed)
      *decomposed = static_cast<int>(h->dd_levels.size());
  });
}

int pmg_dd_slab(pmg_dd h, int local, int which, void **ptr, int64_t *z0, int64_t *nplanes, int64_t *own_lo,
                int64_t *own_hi)
{
  return dd_guard([&] {
    if (!h || local < 0 || local >= static_cast<int>(h->local.size()) || (which != PMG_DD_X && which != PMG_DD_B))
      throw InvalidArg("dd_slab: invalid arguments");
    LevelState &ls = h->local[local]->L[h->finest];
    if (ptr)
      *ptr = ls.a[which == PMG_DD_X ? A_X : A_B];
    if (z0)
      *z0 = ls.slab.e0;
    if (nplanes)
      *nplanes = ls.slab.np();
    if (own_lo)
      *own_lo = ls.slab.plan.own_lo;
    if (own_hi)
      *own_hi = ls.slab.plan.own_hi;
  });
}

int pmg_dd_stream(pmg_dd h, int local, void **stream, int *rank)
{
  return dd_guard([&] {
    if (!h || local < 0 || local >= static_cast<int>(h->local.size()))
      throw InvalidArg("dd_stream: invalid arguments");
    if (stream)
      *stream = h->local[local]->main;
    if (rank)
      *rank = h->local[local]->rank;
  });
}

int pmg_dd_scatter_host(pmg_dd h, int which, const void *global)
{
  return dd_guard([&] {
    if (!h || !global || (which != PMG_DD_X && which != PMG_DD_B))
      throw InvalidArg("dd_scatter_host: invalid arguments");
    sync_all(h);
    scatter_host(h, h->finest, which == PMG_DD_X ? A_X : A_B, global);
  });
}

int pmg_dd_gather_host(pmg_dd h, int which, void *global)
{
  return dd_guard([&] {
    if (!h || !global || (which != PMG_DD_X && which != PMG_DD_B))
      throw InvalidArg("dd_gather_host: invalid arguments");
    sync_all(h);
    const int lev = h->finest;
    const int64_t ps = h->ps(lev);
    for (auto &rp : h->local)
    {
      Rank &r = *rp;
      DevScope g(r.device);
      LevelState &ls = r.L[lev];
      const Plan &p = ls.slab.plan;
      check_cuda(cudaMemcpyAsync(static_cast<char *>(global) + h->bytes(p.own_lo * ps),
                                 ls.a[which == PMG_DD_X ? A_X : A_B] + h->bytes((p.own_lo - ls.slab.e0) * ps),
                                 h->bytes((p.own_hi - p.own_lo + 1) * ps), cudaMemcpyDeviceToHost, r.main),
                 "gather D2H");
      check_cuda(cudaStreamSynchronize(r.main), "sync");
    }
  });
}

int pmg_dd_set_smoothing(pmg_dd h, int pre, int post)
{
  return dd_guard([&] {
    if (!h || pre < 0 || post < 0)
      throw InvalidArg("invalid smoothing counts");
    h->pre = pre;
    h->post = post;
    for (auto &rp : h->local)
      if (rp->root_mg)
        ck(pmg_mg_set_smoothing(rp->root_mg, pre, post), "dd coarse context");
  });
}

// the finest level's smoothing step captured once as one CUDA graph (all
// local ranks on one device: virtual ranks, or one process per GPU): the
// per-colour launches, events, copies / NCCL calls of smooth_level replay
// without host work. The other ranks' streams fork from and join the first
// rank's stream inside the capture.
int pmg_dd_set_graph(pmg_dd h, int enable)
{
  return dd_guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    if (enable && !dd_graphable(h))
      throw InvalidArg("dd_set_graph: the local ranks must share one device");
    h->use_graph = enable != 0;
    if (!h->use_graph)
    {
      DevScope g(h->local[0]->device);
      sync_all(h);
      for (cudaGraphExec_t *e : {&h->smooth_graph, &h->vcycle_graph})
        if (*e)
        {
          cudaGraphExecDestroy(*e);
          *e = nullptr;
        }
    }
  });
}

int pmg_dd_smooth(pmg_dd h)
{
  return dd_guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    if (h->use_graph)
    {
      if (!h->smooth_graph)
        dd_capture(h, h->smooth_graph, [&] { smooth_level(h, h->finest); });
      DevScope g(h->local[0]->device);
      check_cuda(cudaGraphLaunch(h->smooth_graph, h->local[0]->main), "graph launch");
      return;
    }
    smooth_level(h, h->finest);
  });
}

int pmg_dd_v_cycle(pmg_dd h)
{
  return dd_guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    check_vcycle(h, "dd_v_cycle");
    if (h->use_graph)
    {
      if (!h->vcycle_graph)
      {
        // the coarse context's workspaces are settled by one eager cycle
        // first (a capture must not allocate): x is restored afterwards
        vcycle_warm(h);
        dd_capture(h, h->vcycle_graph, [&] { vcycle_finest(h); });
      }
      DevScope g(h->local[0]->device);
      check_cuda(cudaGraphLaunch(h->vcycle_graph, h->local[0]->main), "graph launch");
      return;
    }
    vcycle_finest(h);
  });
}

int pmg_dd_residual_norm(pmg_dd h, double *out)
{
  return dd_guard([&] {
    if (!h || !out)
      throw InvalidArg("dd_residual_norm: invalid arguments");
    check_vcycle(h, "dd_residual_norm");
    residual_finest(h);
    *out = norm_owned(h, A_R);
  });
}

int pmg_dd_full_multigrid(pmg_dd h, const double *const *rhs, double tol, int max_iterations, int *iterations,
                          double *history, int history_cap)
{
  std::vector<double> hist;
  const int st = dd_guard([&] {
    if (!h || !rhs)
      throw InvalidArg("dd_full_multigrid: invalid arguments");
    if (h->dtype != PMG_F64)
      throw InvalidArg("full_multigrid runs in f64 only (multigrid.hpp:80)");
    if (!(tol > 0.0))
      throw InvalidArg("full_multigrid: tol must be positive");
    check_vcycle(h, "dd_full_multigrid");
    for (int li = 0; li < h->finest; ++li)
      if (!rhs[li])
        throw InvalidArg("full_multigrid: need one rhs per level");
    const int F = h->finest;
    sync_all(h);
    // nested iteration (multigrid.cpp:368-377): the agglomerated levels on rank 0
    if (Rank *root = h->find(0))
    {
      DevScope g(root->device);
      for (int l = 1; l <= h->agg; ++l)
      {
        const size_t bytes = h->bytes(h->mz(l) * h->ps(l));
        root->fmg_x[l].ensure(bytes);
        root->fmg_b[l].ensure(bytes);
        check_cuda(cudaMemcpyAsync(root->fmg_b[l].p, rhs[l - 1], bytes, cudaMemcpyHostToDevice, root->main), "H2D");
        if (l == 1)
          ck(pmg_v_cycle(root->root_mg, 0, root->fmg_x[1].p, root->fmg_b[1].p, 0, root->main), "fmg coarse solve");
        else
        {
          ck(pmg_prolongate(pmg_mg_level(root->root_mg, l - 2), pmg_mg_level(root->root_mg, l - 1),
                            root->fmg_x[l - 1].p, root->fmg_x[l].p, 0, root->main),
             "fmg prolongate");
          ck(pmg_v_cycle(root->root_mg, l - 1, root->fmg_x[l].p, root->fmg_b[l].p, 0, root->main), "fmg V-cycle");
        }
      }
      check_cuda(cudaStreamSynchronize(root->main), "sync");
    }
    if (h->dd_levels.empty())
    {
      // every level agglomerated: rank 0's finest iterate into the slabs
      const int64_t ps = h->ps(F), words = h->mz(F) * ps;
      if (Rank *root = h->find(0))
      {
        DevScope g(root->device);
        check_cuda(cudaMemcpyAsync(root->L[F].a[A_XC], root->fmg_x[F].p, h->bytes(words), cudaMemcpyDeviceToDevice,
                                   root->main),
                   "D2D");
      }
      broadcast_from_root(h, F, A_XC, words);
      for (auto &rp : h->local)
      {
        Rank &r = *rp;
        DevScope g(r.device);
        LevelState &ls = r.L[F];
        copy_planes(h, r, ls.a[A_X], ls.slab.e0, r, ls.a[A_XC], 0, ls.slab.e0, ls.slab.np(), ps, r.main);
      }
      scatter_host(h, F, A_B, rhs[F - 1]);
    }
    else
    {
      // decomposed levels, coarsest first: x_l = P x_{l-1}, then one V-cycle
      // (the finest included, as in the reference). A coarser level's x / b
      // are the finer level's x_c / b_c arrays, so x_{l-1} is level l's x_c
      // when level l prolongates it.
      for (auto it = h->dd_levels.rbegin(); it != h->dd_levels.rend(); ++it)
      {
        const int lev = *it, cl = lev - 1;
        scatter_host(h, lev, A_B, rhs[lev - 1]);
        if (!h->is_dd(cl))
        {
          if (Rank *root = h->find(0))
          {
            DevScope g(root->device);
            check_cuda(cudaMemcpyAsync(root->L[lev].a[A_XC], root->fmg_x[cl].p, h->bytes(h->mz(cl) * h->ps(cl)),
                                       cudaMemcpyDeviceToDevice, root->main),
                       "D2D");
          }
          broadcast_from_root(h, lev, A_XC, h->mz(cl) * h->ps(cl));
        }
        else
          halo(h, cl, A_X);
        for (auto &rp : h->local)
        {
          Rank &r = *rp;
          DevScope g(r.device);
          LevelState &ls = r.L[lev];
          check_cuda(cudaMemsetAsync(ls.a[A_X], 0, h->bytes(ls.slab.np() * h->ps(lev)), r.main), "memset");
          int64_t e0c = 0, npc = h->mz(cl);
          if (h->is_dd(cl))
          {
            e0c = r.L[cl].slab.e0;
            npc = r.L[cl].slab.np();
          }
          ck(pmg_prolongate_slab(h->lv(r, cl), ls.lv, ls.a[A_XC], e0c, npc, ls.a[A_X], ls.slab.e0, ls.slab.np(),
                                 ls.slab.plan.lo, ls.slab.plan.hi + 1, 0, r.main),
             "fmg prolongate");
        }
        vcycle_level(h, lev);
      }
    }
    // the while loop on the finest level (multigrid.cpp:381-398)
    const double delta0 = norm_owned(h, A_B);
    hist.push_back(delta0);
    double delta = delta0;
    int its = 0;
    while (delta > tol * delta0)
    {
      if (its >= max_iterations)
        throw DivergenceErr("full_multigrid: no convergence after " + std::to_string(max_iterations) + " V-cycles");
      vcycle_finest(h);
      residual_finest(h);
      delta = norm_owned(h, A_R);
      hist.push_back(delta);
      ++its;
    }
    if (iterations)
      *iterations = its;
  });
  if (history)
    for (int i = 0; i < history_cap && i < static_cast<int>(hist.size()); ++i)
      history[i] = hist[i];
  if (iterations && st == PMG_ERR_DIVERGENCE)
    *iterations = max_iterations;
  return st;
}

int pmg_dd_synchronize(pmg_dd h)
{
  return dd_guard([&] {
    if (!h)
      throw InvalidArg("null handle");
    sync_all(h);
  });
}

}  // extern "C"
