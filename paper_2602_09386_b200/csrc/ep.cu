// Expert-parallel data movement (BASELINE config c5: experts sharded E/n per GPU).
//
// The reference runs every expert in one process (execution.py:85-191); under expert
// parallelism rank r owns experts [r*E_l, (r+1)*E_l) and every rank routes its own batch
// shard.  One step moves, per (source s, owner r):
//   dispatch : h[b] once per (b, r) with U_b meeting r's experts (dedup per destination GPU),
//              plus the union-mask words of r's experts -> the owner expands to local rows
//   return   : the head projections P (T floats) of every (b, e) row, in the source's plan order
//   backward : the row coefficients C (T bf16) of every (b, e) row to the owner, and the
//              per-instance input gradient sum over r's experts back to the source.
// All buffers are fixed-slot (slot = worst case per peer) so counts stay on the device and the
// step has no host sync; the transports (NCCL all-to-all, or the peer-memory put in
// smes_ep_put_slots) move the slots.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstring>

#include "ptx.cuh"
#include "smes_capi.h"

namespace smes {

// --- dispatch pack: block r compacts the instances whose union meets owner r's mask words
__global__ void __launch_bounds__(1024) ep_pack_index_kernel(int B, int EW, const uint32_t* __restrict__ umask,
                                                             int wpr, int32_t* __restrict__ idx,
                                                             int32_t* __restrict__ pos, int32_t* __restrict__ cnt,
                                                             uint32_t* __restrict__ mask_out) {
  pdl_wait();
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int r = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    bool pred = false;
    if (b < B)
      for (int w = 0; w < wpr; ++w) pred |= umask[(size_t)b * EW + r * wpr + w] != 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, pred);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int off = base_s;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    const int p = off + __popc(bal & ((1u << lane) - 1u));
    if (b < B) {
      pos[(size_t)r * B + b] = pred ? p : -1;
      if (pred) {
        idx[(size_t)r * B + p] = b;
        for (int w = 0; w < wpr; ++w)
          mask_out[((size_t)r * B + p) * wpr + w] = umask[(size_t)b * EW + r * wpr + w];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += warp_tot[w];
      base_s += t;
    }
    __syncthreads();
  }
  const int n = base_s;
  if (threadIdx.x == 0) cnt[r] = n;
  // empty slots carry zero masks: the owner's plan skips them
  for (size_t i = (size_t)n * wpr + threadIdx.x; i < (size_t)B * wpr; i += blockDim.x)
    mask_out[(size_t)r * B * wpr + i] = 0u;
}

// h_out[r][i] = h[idx[r][i]] for i < cnt[r]  (16-byte vectors)
__global__ void ep_pack_rows_kernel(int B, int d, const int32_t* __restrict__ idx, const int32_t* __restrict__ cnt,
                                    const __nv_bfloat16* __restrict__ h, long ldh, __nv_bfloat16* __restrict__ out) {
  pdl_wait();
  const int r = blockIdx.y;
  const int vec = d / 8;
  const long n = (long)cnt[r] * vec;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long row = i / vec, c = (i - row * vec) * 8;
    const int b = idx[(size_t)r * B + row];
    *reinterpret_cast<uint4*>(out + ((size_t)r * B + row) * d + c) =
        *reinterpret_cast<const uint4*>(h + (size_t)b * ldh + c);
  }
}

// --- segment tables between a packed (expert-major, padded) layout and per-peer slots.
// seg_tab[(s*E_l + e)*3 + {0,1,2}] = {packed row, slot row, rows}
//   owner  (mode 0): cnt[s][e] rows of source s for local expert e; sources are interleaved in
//                    source order inside the owner's segment e starting at seg_pad[e]
//   source (mode 1): cnt[r][e] = loads of owner r's e-th expert, packed at seg_pad[r*E_l + e]
__global__ void ep_segments_kernel(int mode, int n, int El, const int32_t* __restrict__ cnt,
                                   const int32_t* __restrict__ seg_pad, long slot_rows, int32_t* __restrict__ tab) {
  pdl_wait();
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int slot_off = 0;
  for (int e = 0; e < El; ++e) {
    int packed;
    if (mode == 0) {
      packed = seg_pad[e];
      for (int s2 = 0; s2 < s; ++s2) packed += cnt[s2 * El + e];
    } else {
      packed = seg_pad[s * El + e];
    }
    const int c = cnt[s * El + e];
    int32_t* t = tab + ((size_t)s * El + e) * 3;
    t[0] = packed;
    t[1] = (int)(s * slot_rows) + slot_off;
    t[2] = c;
    slot_off += c;
  }
}

// dir 0: packed -> slots (gather), dir 1: slots -> packed (scatter); one block per segment
__global__ void ep_copy_rows_kernel(int dir, const int32_t* __restrict__ tab, const uint8_t* __restrict__ src,
                                    long src_ld, uint8_t* __restrict__ dst, long dst_ld, int row_bytes) {
  pdl_wait();
  const int32_t* t = tab + (size_t)blockIdx.x * 3;
  const long packed = t[0], slot = t[1];
  const int rows = t[2];
  const long s0 = dir == 0 ? packed : slot, d0 = dir == 0 ? slot : packed;
  const int vec = row_bytes / 16;
  for (long i = threadIdx.x; i < (long)rows * vec; i += blockDim.x) {
    const long r = i / vec, c = (i - r * vec) * 16;
    *reinterpret_cast<uint4*>(dst + (d0 + r) * dst_ld + c) = *reinterpret_cast<const uint4*>(src + (s0 + r) * src_ld + c);
  }
}

// d_hidden[b] = dh_router[b] + sum_r dh_recv[r][pos[r][b]]   (fixed owner order)
__global__ void ep_combine_dh_kernel(int B, int d, int n, long slot_rows, const int32_t* __restrict__ pos,
                                     const float* __restrict__ dh_recv, const float* __restrict__ dh_router,
                                     float* __restrict__ out) {
  pdl_wait();
  const int b = blockIdx.x;
  for (int c = threadIdx.x * 4; c < d; c += blockDim.x * 4) {
    float4 acc = dh_router ? *reinterpret_cast<const float4*>(dh_router + (size_t)b * d + c) : make_float4(0, 0, 0, 0);
    for (int r = 0; r < n; ++r) {
      const int p = pos[(size_t)r * B + b];
      if (p >= 0) {
        const float4 v = *reinterpret_cast<const float4*>(dh_recv + ((size_t)r * slot_rows + p) * d + c);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      }
    }
    *reinterpret_cast<float4*>(out + (size_t)b * d + c) = acc;
  }
}

// capacity guard on the owner's plan: if the padded rows exceed the workspace, flag it and
// empty the plan (no kernel downstream touches rows beyond the workspace)
__global__ void ep_capacity_guard_kernel(int E, long cap, const int32_t* __restrict__ totals,
                                         int32_t* __restrict__ seg_pad, int32_t* __restrict__ loads,
                                         uint32_t* __restrict__ umask, long n_mask_words, int32_t* __restrict__ usize,
                                         long n_inst, int32_t* __restrict__ flag) {
  pdl_wait();
  const bool over = (long)totals[1] > cap;
  if (!over) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) *flag = 1;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n_mask_words; i += (long)gridDim.x * blockDim.x)
    umask[i] = 0u;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n_inst; i += (long)gridDim.x * blockDim.x)
    usize[i] = 0;
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e <= E; e += blockDim.x) {
      seg_pad[e] = 0;
      if (e < E) loads[e] = 0;
    }
}

// peer-memory transport: rank `self` writes slot r of its send buffer into slot `self` of rank r's
// receive buffer (peer pointers from CUDA IPC), then raises its flag in every peer's flag array.
// rows_used[r] (device) bounds the bytes actually moved.
struct PutArgs {
  int n, self;
  const uint8_t* send;              // (n, slot_bytes)
  long slot_bytes;
  long row_bytes;
  const int32_t* rows_used;         // (n) rows of each slot to move, or null (whole slot)
  uint8_t* const* peer_recv;        // (n) receive buffers of every rank (own included)
};

__global__ void ep_put_kernel(PutArgs a) {
  pdl_wait();
  const int r = blockIdx.y;
  const long bytes = a.rows_used ? (long)a.rows_used[r] * a.row_bytes : a.slot_bytes;
  const uint8_t* src = a.send + (long)r * a.slot_bytes;
  uint8_t* dst = a.peer_recv[r] + (long)a.self * a.slot_bytes;
  for (long i = (blockIdx.x * (long)blockDim.x + threadIdx.x) * 16; i < bytes; i += (long)gridDim.x * blockDim.x * 16)
    *reinterpret_cast<uint4*>(dst + i) = *reinterpret_cast<const uint4*>(src + i);
}

__global__ void ep_signal_kernel(int n, int self, int32_t* const* peer_flags, int32_t epoch) {
  pdl_wait();
  // publish: every put of this rank is visible system-wide before the flag
  __threadfence_system();
  const int r = threadIdx.x;
  if (r < n) {
    volatile int32_t* f = peer_flags[r] + self;
    *f = epoch;
  }
}

__global__ void ep_wait_kernel(int n, volatile int32_t* my_flags, int32_t epoch) {
  pdl_wait();
  const int r = threadIdx.x;
  if (r < n)
    while (my_flags[r] < epoch) {
    }
  __threadfence_system();
}


// ---------------------------------------------------------------- fused pack + put (peer memory)
// The dispatch writes every packed row straight into slot `self` of the owner's receive buffer
// (peer pointers from CUDA IPC: stores travel over NVLink), so no send buffer and no separate
// all-to-all pass exist.  Same compaction order as ep_pack (instances ascending per owner).
__global__ void __launch_bounds__(1024) ep_pack_index_put_kernel(int B, int EW, const uint32_t* __restrict__ umask,
                                                                 int wpr, int self, int32_t* __restrict__ idx,
                                                                 int32_t* __restrict__ pos, int32_t* __restrict__ cnt,
                                                                 uint32_t* const* __restrict__ peer_mask) {
  pdl_wait();
  __shared__ int warp_tot[32];
  __shared__ int base_s;
  const int r = blockIdx.x;
  uint32_t* mask_out = peer_mask[r] + (size_t)self * B * wpr;     // slot `self` of owner r
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) base_s = 0;
  __syncthreads();
  for (int b0 = 0; b0 < B; b0 += 1024) {
    const int b = b0 + threadIdx.x;
    bool pred = false;
    if (b < B)
      for (int w = 0; w < wpr; ++w) pred |= umask[(size_t)b * EW + r * wpr + w] != 0u;
    const uint32_t bal = __ballot_sync(0xffffffffu, pred);
    if (lane == 0) warp_tot[warp] = __popc(bal);
    __syncthreads();
    int off = base_s;
    for (int w = 0; w < warp; ++w) off += warp_tot[w];
    const int p = off + __popc(bal & ((1u << lane) - 1u));
    if (b < B) {
      pos[(size_t)r * B + b] = pred ? p : -1;
      if (pred) {
        idx[(size_t)r * B + p] = b;
        for (int w = 0; w < wpr; ++w) mask_out[(size_t)p * wpr + w] = umask[(size_t)b * EW + r * wpr + w];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += warp_tot[w];
      base_s += t;
    }
    __syncthreads();
  }
  const int n = base_s;
  if (threadIdx.x == 0) cnt[r] = n;
  for (size_t i = (size_t)n * wpr + threadIdx.x; i < (size_t)B * wpr; i += blockDim.x) mask_out[i] = 0u;
}

__global__ void ep_pack_rows_put_kernel(int B, int d, int self, const int32_t* __restrict__ idx,
                                        const int32_t* __restrict__ cnt, const __nv_bfloat16* __restrict__ h, long ldh,
                                        __nv_bfloat16* const* __restrict__ peer_h) {
  pdl_wait();
  const int r = blockIdx.y;
  __nv_bfloat16* out = peer_h[r] + (size_t)self * B * d;
  const int vec = d / 8;
  const long n = (long)cnt[r] * vec;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
    const long row = i / vec, c = (i - row * vec) * 8;
    const int b = idx[(size_t)r * B + row];
    *reinterpret_cast<uint4*>(out + row * d + c) = *reinterpret_cast<const uint4*>(h + (size_t)b * ldh + c);
  }
}

// gather rows per segment straight into the destination peer's slot `self`:
// segment i belongs to peer s = i / El; its slot row (tab[1]) is relative to s * slot_rows locally
__global__ void ep_copy_rows_put_kernel(const int32_t* __restrict__ tab, int El, long slot_rows, int self,
                                        const uint8_t* __restrict__ src, long src_ld, uint8_t* const* __restrict__ peer,
                                        long dst_ld, int row_bytes) {
  pdl_wait();
  const int i = blockIdx.x;
  const int s = i / El;
  const int32_t* t = tab + (size_t)i * 3;
  const long packed = t[0], drow = t[1] - (long)s * slot_rows + (long)self * slot_rows;
  const int rows = t[2];
  uint8_t* dst = peer[s];
  const int vec = row_bytes / 16;
  for (long k = threadIdx.x; k < (long)rows * vec; k += blockDim.x) {
    const long r = k / vec, c = (k - r * vec) * 16;
    *reinterpret_cast<uint4*>(dst + (drow + r) * dst_ld + c) = *reinterpret_cast<const uint4*>(src + (packed + r) * src_ld + c);
  }
}

}  // namespace smes

using namespace smes;

static int launch_ok(const char* what) {
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SMES_OK : set_error(SMES_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

extern "C" {

int smes_ep_pack(int B, int EW, const uint32_t* umask, int n, int wpr, const void* h, long ldh, int d, int32_t* idx,
                 int32_t* pos, int32_t* cnt, uint32_t* mask_out, void* h_out, void* stream) {
  if (n < 1 || n > 64 || wpr < 1 || n * wpr > EW) return set_error(SMES_ERR_SHAPE, "ep_pack: n=%d wpr=%d EW=%d", n, wpr, EW);
  if (d % 8) return set_error(SMES_ERR_SHAPE, "ep_pack: d=%d must be a multiple of 8", d);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  smes_launch(ep_pack_index_kernel, n, 1024, 0, st, B, EW, umask, wpr, idx, pos, cnt, mask_out);
  if (h != nullptr) {
    dim3 g(296, n);
    smes_launch(ep_pack_rows_kernel, g, 256, 0, st, B, d, idx, cnt, reinterpret_cast<const __nv_bfloat16*>(h), ldh,
                                          reinterpret_cast<__nv_bfloat16*>(h_out));
  }
  return launch_ok("ep_pack");
}

int smes_ep_segments(int mode, int n, int El, const int32_t* cnt, const int32_t* seg_pad, long slot_rows,
                     int32_t* tab, void* stream) {
  if (mode != 0 && mode != 1) return set_error(SMES_ERR_CONFIG, "ep_segments: mode %d", mode);
  smes_launch(ep_segments_kernel, (n + 63) / 64, 64, 0, reinterpret_cast<cudaStream_t>(stream), mode, n, El, cnt, seg_pad,
                                                                                     slot_rows, tab);
  return launch_ok("ep_segments");
}

int smes_ep_copy_rows(int nseg, const int32_t* tab, int dir, const void* src, long src_ld_bytes, void* dst,
                      long dst_ld_bytes, int row_bytes, void* stream) {
  if (row_bytes % 16 || src_ld_bytes % 16 || dst_ld_bytes % 16)
    return set_error(SMES_ERR_SHAPE, "ep_copy_rows: rows must be 16-byte multiples (row %d, ld %ld/%ld)", row_bytes,
                     src_ld_bytes, dst_ld_bytes);
  if (nseg == 0) return SMES_OK;
  smes_launch(ep_copy_rows_kernel, nseg, 256, 0, reinterpret_cast<cudaStream_t>(stream), 
      dir, tab, reinterpret_cast<const uint8_t*>(src), src_ld_bytes, reinterpret_cast<uint8_t*>(dst), dst_ld_bytes,
      row_bytes);
  return launch_ok("ep_copy_rows");
}

int smes_ep_combine_dh(int B, int d, int n, long slot_rows, const int32_t* pos, const float* dh_recv,
                       const float* dh_router, float* out, void* stream) {
  if (d % 4) return set_error(SMES_ERR_SHAPE, "ep_combine_dh: d=%d", d);
  smes_launch(ep_combine_dh_kernel, B, 256, 0, reinterpret_cast<cudaStream_t>(stream), B, d, n, slot_rows, pos, dh_recv,
                                                                            dh_router, out);
  return launch_ok("ep_combine_dh");
}

int smes_ep_capacity_guard(int E, long cap, const int32_t* totals, int32_t* seg_pad, int32_t* loads, uint32_t* umask,
                           long n_mask_words, int32_t* usize, long n_inst, int32_t* flag, void* stream) {
  smes_launch(ep_capacity_guard_kernel, 64, 256, 0, reinterpret_cast<cudaStream_t>(stream), E, cap, totals, seg_pad, loads,
                                                                                 umask, n_mask_words, usize, n_inst,
                                                                                 flag);
  return launch_ok("ep_capacity_guard");
}


int smes_ep_pack_put(int B, int EW, const uint32_t* umask, int n, int wpr, const void* h, long ldh, int d, int self,
                     int32_t* idx, int32_t* pos, int32_t* cnt, void* const* peer_mask_recv,
                     void* const* peer_h_recv, void* stream) {
  if (n < 1 || n > 64 || wpr < 1 || n * wpr > EW) return set_error(SMES_ERR_SHAPE, "ep_pack_put: n=%d wpr=%d EW=%d", n, wpr, EW);
  if (d % 8) return set_error(SMES_ERR_SHAPE, "ep_pack_put: d=%d must be a multiple of 8", d);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  smes_launch(ep_pack_index_put_kernel, n, 1024, 0, st, B, EW, umask, wpr, self, idx, pos, cnt,
                                              reinterpret_cast<uint32_t* const*>(peer_mask_recv));
  dim3 g(296, n);
  smes_launch(ep_pack_rows_put_kernel, g, 256, 0, st, B, d, self, idx, cnt, reinterpret_cast<const __nv_bfloat16*>(h), ldh,
                                            reinterpret_cast<__nv_bfloat16* const*>(peer_h_recv));
  return launch_ok("ep_pack_put");
}

int smes_ep_copy_rows_put(int nseg, const int32_t* tab, int El, long slot_rows, int self, const void* src,
                          long src_ld_bytes, void* const* peer_dst, long dst_ld_bytes, int row_bytes, void* stream) {
  if (row_bytes % 16 || src_ld_bytes % 16 || dst_ld_bytes % 16)
    return set_error(SMES_ERR_SHAPE, "ep_copy_rows_put: rows must be 16-byte multiples");
  if (nseg == 0) return SMES_OK;
  smes_launch(ep_copy_rows_put_kernel, nseg, 256, 0, reinterpret_cast<cudaStream_t>(stream), 
      tab, El, slot_rows, self, reinterpret_cast<const uint8_t*>(src), src_ld_bytes,
      reinterpret_cast<uint8_t* const*>(peer_dst), dst_ld_bytes, row_bytes);
  return launch_ok("ep_copy_rows_put");
}

int smes_ep_put_slots(int n, int self, const void* send, long slot_bytes, long row_bytes, const int32_t* rows_used,
                      void* const* peer_recv_dev, void* stream) {
  if (slot_bytes % 16 || row_bytes % 16) return set_error(SMES_ERR_SHAPE, "ep_put: slot/row bytes must be 16-aligned");
  PutArgs a{n, self, reinterpret_cast<const uint8_t*>(send), slot_bytes, row_bytes, rows_used,
            reinterpret_cast<uint8_t* const*>(peer_recv_dev)};
  dim3 g(148, n);
  smes_launch(ep_put_kernel, g, 512, 0, reinterpret_cast<cudaStream_t>(stream), a);
  return launch_ok("ep_put");
}

int smes_ep_signal_wait(int n, int self, void* const* peer_flags_dev, int32_t* my_flags, int epoch, void* stream) {
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  smes_launch(ep_signal_kernel, 1, 64, 0, st, n, self, reinterpret_cast<int32_t* const*>(peer_flags_dev), epoch);
  smes_launch(ep_wait_kernel, 1, 64, 0, st, n, my_flags, epoch);
  return launch_ok("ep_signal_wait");
}

// CUDA IPC helpers for the peer-memory transport (handles travel through torch.distributed)
// The IPC handle names the whole cudaMalloc allocation that contains dev_ptr, and the peer's
// cudaIpcOpenMemHandle returns that allocation's BASE.  Tensors from a caching allocator sit at an
// offset inside a larger segment, so the offset travels with the handle (offset_out) and the peer
// adds it to the mapped base (smes_ipc_open).
int smes_ipc_handle(void* dev_ptr, void* handle_out /* 64 bytes */, long* offset_out) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, dev_ptr);
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  static GetRange get_range = nullptr;
  if (get_range == nullptr) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fp == nullptr)
      return set_error(SMES_ERR_CUDA, "cuMemGetAddressRange entry point unavailable");
    get_range = reinterpret_cast<GetRange>(fp);
  }
  unsigned long long base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (unsigned long long)dev_ptr) != 0)
    return set_error(SMES_ERR_CUDA, "cuMemGetAddressRange failed for %p", dev_ptr);
  memcpy(handle_out, &h, sizeof(h));
  if (offset_out) *offset_out = (long)((unsigned long long)dev_ptr - base);
  return SMES_OK;
}

int smes_ipc_open(const void* handle /* 64 bytes */, void** dev_ptr_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  return SMES_OK;
}

int smes_ipc_close(void* dev_ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) return set_error(SMES_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return SMES_OK;
}

}  // extern "C"
