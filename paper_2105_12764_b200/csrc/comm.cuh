// Block-sharded multi-GPU support: the visible-device
// count for embarrassing_decompose's worker -> GPU map, the cooperative slab
// schedule (for CommReport::idle), per-block metadata records and their one
// NCCL all-gather.  The data path has no collective: every rank refactors
// whole blocks (parallel_impl.hpp:810-847); the gather only publishes where
// each block's classes are and how large they are.
#pragma once

#include <nccl.h>
#include <zlib.h>

struct mgrg_comm {
  ncclComm_t nc = nullptr;
  int nranks = 0, rank = 0, device = 0;
  cudaStream_t stream = nullptr;
  void *d_buf = nullptr;
  size_t cap = 0; // bytes of d_buf
};

namespace {

mgrg_status nccl_fail(ncclResult_t r, const char *what) {
  return fail(MGRG_NCCL_ERROR, std::string(what) + ": " + ncclGetErrorString(r));
}

} // namespace

extern "C" {

mgrg_status mgrg_device_count(int32_t *count) {
  g_last_error.clear();
  if (!count)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(MGRG_CUDA_ERROR, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  }
  *count = n;
  return MGRG_OK;
}

mgrg_status mgrg_coop_schedule(const mgrg_plan *p, int32_t workers, int32_t *q,
                               uint64_t *bounds) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!q || workers < 1)
    return fail(MGRG_INVALID_ARGUMENT, "null q or workers < 1");
  *q = 0;
  const int L = p->H.L;
  if (workers == 1 || p->H.nd != 3 || p->gen || !p->lean)
    return MGRG_OK;
  std::vector<std::array<uint64_t, 3>> ls;
  for (int l = 0; l <= L; ++l)
    ls.push_back({p->H.ext[l][0], p->H.ext[l][1], p->H.ext[l][2]});
  const int qq = coop_depth(ls, workers); // the runtime's rule (coop_host.cuh)
  *q = qq;
  if (qq > 0 && bounds) {
    const uint64_t n2 = ls[L][2], units = (n2 - 1) >> qq, W = uint64_t(workers);
    for (uint64_t r = 0; r < W; ++r)
      bounds[r] = ((units / W) * r + std::min<uint64_t>(r, units % W)) << qq;
    bounds[W] = n2 - 1;
  }
  return MGRG_OK;
}

mgrg_status mgrg_block_meta_fill(mgrg_plan *p, const void *d_classes, int64_t block_id,
                                 int32_t rank, const uint64_t *origin, double dec_ms,
                                 double rec_ms, mgrg_block_meta *m, void *stream) {
  g_last_error.clear();
  if (mgrg_status st = check_plan(p))
    return st;
  if (!d_classes || !m)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  const int L = p->H.L;
  if (L + 1 > MGRG_MAX_CLASSES)
    return fail(MGRG_UNSUPPORTED, "more classes than MGRG_MAX_CLASSES");
  std::memset(m, 0, sizeof(*m));
  m->block_id = block_id;
  m->rank = rank;
  m->dtype = int32_t(p->esize);
  m->ndims = p->H.nd;
  m->levels = L;
  for (int d = 0; d < p->H.nd; ++d) {
    m->shape[d] = p->H.shape[d];
    m->origin[d] = origin ? origin[d] : 0;
  }
  for (int l = 0; l <= L; ++l)
    m->class_bytes[l] = class_count(p, l) * p->esize;
  if (mgrg_status st = mgrg_class_crc32(p, d_classes, L, m->class_crc32, stream))
    return st;
  uint8_t le[4 * MGRG_MAX_CLASSES];
  for (int l = 0; l <= L; ++l)
    for (int b = 0; b < 4; ++b)
      le[4 * l + b] = uint8_t(m->class_crc32[l] >> (8 * b));
  m->checksum = uint32_t(::crc32(0L, le, uInt(4 * (L + 1))));
  m->decompose_ms = dec_ms;
  m->recompose_ms = rec_ms;
  return MGRG_OK;
}

mgrg_status mgrg_comm_unique_id(uint8_t id[MGRG_COMM_ID_BYTES]) {
  g_last_error.clear();
  static_assert(sizeof(ncclUniqueId) == MGRG_COMM_ID_BYTES, "NCCL unique id size");
  if (!id)
    return fail(MGRG_INVALID_ARGUMENT, "null argument");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess)
    return nccl_fail(r, "ncclGetUniqueId");
  std::memcpy(id, &u, sizeof(u));
  return MGRG_OK;
}

mgrg_status mgrg_comm_init(const uint8_t id[MGRG_COMM_ID_BYTES], int32_t nranks, int32_t rank,
                           int32_t device, mgrg_comm **out) {
  g_last_error.clear();
  if (!id || !out || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(MGRG_INVALID_ARGUMENT, "bad communicator arguments");
  *out = nullptr;
  DeviceGuard guard(device);
  auto c = std::make_unique<mgrg_comm>();
  c->nranks = nranks;
  c->rank = rank;
  c->device = device;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclResult_t r = ncclCommInitRank(&c->nc, nranks, u, rank);
  if (r != ncclSuccess)
    return nccl_fail(r, "ncclCommInitRank");
  cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    ncclCommDestroy(c->nc);
    return fail(MGRG_CUDA_ERROR, std::string("cudaStreamCreate: ") + cudaGetErrorString(e));
  }
  *out = c.release();
  return MGRG_OK;
}

mgrg_status mgrg_comm_destroy(mgrg_comm *c) {
  g_last_error.clear();
  if (!c)
    return MGRG_OK;
  DeviceGuard guard(c->device);
  if (c->d_buf)
    cudaFree(c->d_buf);
  if (c->stream)
    cudaStreamDestroy(c->stream);
  ncclResult_t r = c->nc ? ncclCommDestroy(c->nc) : ncclSuccess;
  delete c;
  return r == ncclSuccess ? MGRG_OK : nccl_fail(r, "ncclCommDestroy");
}

mgrg_status mgrg_comm_size(const mgrg_comm *c, int32_t *nranks, int32_t *rank) {
  g_last_error.clear();
  if (!c)
    return fail(MGRG_INVALID_ARGUMENT, "null communicator");
  if (nranks)
    *nranks = c->nranks;
  if (rank)
    *rank = c->rank;
  return MGRG_OK;
}

mgrg_status mgrg_comm_allgather_block_meta(mgrg_comm *c, const mgrg_block_meta *mine,
                                           int32_t per_rank, mgrg_block_meta *all,
                                           void *stream) {
  g_last_error.clear();
  if (!c || !all || per_rank < 0 || (per_rank > 0 && !mine))
    return fail(MGRG_INVALID_ARGUMENT, "bad all-gather arguments");
  DeviceGuard guard(c->device);
  const size_t one = size_t(per_rank) * sizeof(mgrg_block_meta);
  const size_t need = one * size_t(c->nranks + 1); // [mine | all]
  if (need > c->cap) {
    if (c->d_buf)
      cudaFree(c->d_buf);
    c->d_buf = nullptr;
    c->cap = 0;
    cudaError_t e = cudaMalloc(&c->d_buf, need);
    if (e != cudaSuccess)
      return fail(MGRG_OUT_OF_MEMORY, std::string("meta buffer: ") + cudaGetErrorString(e));
    c->cap = need;
  }
  if (per_rank == 0)
    return MGRG_OK;
  cudaStream_t s = c->stream;
  if (stream) { // order after the caller's work on its stream
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev, static_cast<cudaStream_t>(stream)));
    CUDA_TRY(cudaStreamWaitEvent(s, ev, 0));
    cudaEventDestroy(ev);
  }
  uint8_t *d_mine = static_cast<uint8_t *>(c->d_buf), *d_all = d_mine + one;
  CUDA_TRY(cudaMemcpyAsync(d_mine, mine, one, cudaMemcpyHostToDevice, s));
  ncclResult_t r = ncclAllGather(d_mine, d_all, one, ncclUint8, c->nc, s);
  if (r != ncclSuccess)
    return nccl_fail(r, "ncclAllGather");
  CUDA_TRY(cudaMemcpyAsync(all, d_all, one * size_t(c->nranks), cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return MGRG_OK;
}

} // extern "C"
