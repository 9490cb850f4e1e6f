// Symmetric device buffers: the B200 UnboundBuffer (SPEC.md:183-186,
// PAPER.md:321). One VMM allocation per rank, exported as a POSIX fd,
// imported and mapped by every peer (unicast NVLink path for the SM and CE
// rails) and bound to an NVSwitch multicast object (NVLS rail).
#include <unistd.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "internal.h"

namespace nz {

namespace {

CUmemAllocationProp deviceProp(int device) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return prop;
}

char* mapHandle(CUmemGenericAllocationHandle h, size_t size, size_t align, int device) {
  CUdeviceptr va = 0;
  NZ_CU(NZ_DRV(cuMemAddressReserve)(&va, size, align, 0, 0));
  NZ_CU(NZ_DRV(cuMemMap)(va, size, 0, h, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  NZ_CU(NZ_DRV(cuMemSetAccess)(va, size, &acc, 1));
  return reinterpret_cast<char*>(va);
}

void unmap(char* p, size_t size) {
  if (!p) return;
  const CUdeviceptr va = reinterpret_cast<CUdeviceptr>(p);
  NZ_DRV(cuMemUnmap)(va, size);
  NZ_DRV(cuMemAddressFree)(va, size);
}

}  // namespace

nz_buf* allocSymmetric(nz_comm* c, size_t bytes) {
  if (bytes == 0) fail(NZ_ERR_INVALID, "buffer size must be positive");
  NZ_CUDA(cudaSetDevice(c->device));
  auto* b = new nz_buf();
  b->comm = c;
  b->size = bytes;
  b->ptrs.assign(c->world, nullptr);
  b->imported.assign(c->world, 0);
  try {
    CUmemAllocationProp prop = deviceProp(c->device);
    size_t gran = 0;
    NZ_CU(NZ_DRV(cuMemGetAllocationGranularity)(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmulticastObjectProp mprop{};
    if (c->multicast) {
      mprop.numDevices = static_cast<unsigned>(c->world);
      mprop.size = bytes;
      mprop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
      size_t mg = 0;
      NZ_CU(NZ_DRV(cuMulticastGetGranularity)(&mg, &mprop, CU_MULTICAST_GRANULARITY_MINIMUM));
      gran = std::max(gran, mg);
    }
    b->mapped = (bytes + gran - 1) / gran * gran;
    if (getenv("NEZHA_DEBUG")) {
      size_t fr = 0, tot = 0;
      cudaMemGetInfo(&fr, &tot);
      fprintf(stderr, "[nezha] rank %d alloc %zu -> %zu (gran %zu) free %zu / %zu MiB\n", c->rank, bytes, b->mapped,
              gran, fr >> 20, tot >> 20);
    }
    NZ_CU(NZ_DRV(cuMemCreate)(&b->local, b->mapped, &prop, 0));
    b->ptrs[c->rank] = mapHandle(b->local, b->mapped, gran, c->device);

    if (c->loop) {
      // Virtual ranks share this process's address space and GPU: the peers'
      // mappings are their own, passed by pointer (no import, no multicast).
      struct {
        uint64_t mapped;
        uint64_t va;
      } mine{b->mapped, reinterpret_cast<uint64_t>(b->ptrs[c->rank])};
      const auto msgs = exchange(c, &mine, sizeof(mine), {});
      for (int p = 0; p < c->world; ++p) {
        decltype(mine) theirs{};
        memcpy(&theirs, msgs[p].data.data(), sizeof(theirs));
        if (theirs.mapped != b->mapped) fail(NZ_ERR_INVALID, "asymmetric buffer allocation");
        b->ptrs[p] = reinterpret_cast<char*>(theirs.va);
      }
    } else if (c->world > 1) {
      int fd = -1;
      NZ_CU(NZ_DRV(cuMemExportToShareableHandle)(&fd, b->local, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
      uint64_t mine = b->mapped;
      auto msgs = exchange(c, &mine, sizeof(mine), {fd});
      close(fd);
      for (int p = 0; p < c->world; ++p) {
        if (p == c->rank) continue;
        uint64_t theirs = 0;
        memcpy(&theirs, msgs[p].data.data(), sizeof(theirs));
        if (theirs != b->mapped || msgs[p].fds.size() != 1) fail(NZ_ERR_INVALID, "asymmetric buffer allocation");
        const int pfd = msgs[p].fds[0];
        CUresult r = NZ_DRV(cuMemImportFromShareableHandle)(&b->imported[p], reinterpret_cast<void*>(static_cast<intptr_t>(pfd)),
                                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
        close(pfd);
        NZ_CU(r);
        b->ptrs[p] = mapHandle(b->imported[p], b->mapped, gran, c->device);
      }

      if (c->multicast) {
        mprop.size = b->mapped;
        int mfd = -1;
        if (c->rank == 0) {
          NZ_CU(NZ_DRV(cuMulticastCreate)(&b->mc, &mprop));
          NZ_CU(NZ_DRV(cuMemExportToShareableHandle)(&mfd, b->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
        }
        std::vector<int> send;
        if (c->rank == 0) send.push_back(mfd);
        auto mm = exchange(c, nullptr, 0, send);
        if (mfd >= 0) close(mfd);
        if (c->rank != 0) {
          if (mm[0].fds.size() != 1) fail(NZ_ERR_SYSTEM, "multicast handle missing from rank 0");
          const int rfd = mm[0].fds[0];
          for (size_t i = 1; i < mm.size(); ++i)
            for (int f : mm[i].fds) close(f);
          CUresult r = NZ_DRV(cuMemImportFromShareableHandle)(&b->mc, reinterpret_cast<void*>(static_cast<intptr_t>(rfd)),
                                                      CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
          close(rfd);
          NZ_CU(r);
        }
        CUdevice dev;
        NZ_CU(NZ_DRV(cuDeviceGet)(&dev, c->device));
        NZ_CU(NZ_DRV(cuMulticastAddDevice)(b->mc, dev));
        // Blocks until every device of the team has been added.
        NZ_CU(NZ_DRV(cuMulticastBindMem)(b->mc, 0, b->local, 0, b->mapped, 0));
        b->mc_ptr = mapHandle(b->mc, b->mapped, gran, c->device);
        exchange(c, nullptr, 0, {});  // bound everywhere before any multimem access
      }
    }
  } catch (...) {
    freeSymmetric(b, false);  // peers may have failed elsewhere: no rendezvous
    throw;
  }
  return b;
}

void freeSymmetric(nz_buf* b, bool collective) {
  if (!b) return;
  nz_comm* c = b->comm;
  cudaSetDevice(c->device);
  if (collective && c->world > 1) {
    // Peers read and write this memory over NVLink (or, for virtual ranks, in
    // the same process): unmap it only once no kernel of any rank can still
    // touch it — even after a failed op, whose late peers keep running until
    // their own budgets expire. This rank's kernels first, then every peer's
    // (all ranks free in the same order).
    cudaDeviceSynchronize();
    try {
      exchange(c, nullptr, 0, {});
    } catch (...) {
    }
  }
  cudaDeviceSynchronize();
  if (b->mc_ptr) unmap(b->mc_ptr, b->mapped);
  if (b->mc) {
    CUdevice dev;
    if (NZ_DRV(cuDeviceGet)(&dev, c->device) == CUDA_SUCCESS) NZ_DRV(cuMulticastUnbind)(b->mc, dev, 0, b->mapped);
    NZ_DRV(cuMemRelease)(b->mc);
  }
  for (int p = 0; p < static_cast<int>(b->ptrs.size()); ++p)
    if (!c->loop || p == c->rank) unmap(b->ptrs[p], b->mapped);
  for (auto h : b->imported)
    if (h) NZ_DRV(cuMemRelease)(h);
  if (b->local) NZ_DRV(cuMemRelease)(b->local);
  delete b;
}

}  // namespace nz

using nz::fail;
using nz::guarded;

extern "C" {

int nz_buffer_alloc(nz_comm_t* comm, size_t bytes, nz_buf_t** out) {
  return guarded([&] {
    if (!comm || !out) fail(NZ_ERR_INVALID, "null argument");
    *out = nz::allocSymmetric(comm, bytes);
  });
}

int nz_buffer_free(nz_buf_t* buf) {
  return guarded([&] {
    if (!buf) return;
    nz::freeSymmetric(buf);  // collective: nobody unmaps while a peer may still touch the memory
  });
}

void* nz_buffer_ptr(const nz_buf_t* b) { return b ? b->ptrs[b->comm->rank] : nullptr; }
void* nz_buffer_peer_ptr(const nz_buf_t* b, int rank) {
  if (!b || rank < 0 || rank >= b->comm->world) return nullptr;
  return b->ptrs[rank];
}
void* nz_buffer_mc_ptr(const nz_buf_t* b) { return b ? b->mc_ptr : nullptr; }
size_t nz_buffer_size(const nz_buf_t* b) { return b ? b->size : 0; }

namespace {
void copyChecked(const nz_buf_t* b, uint64_t offset, uint64_t bytes) {
  if (!b) fail(NZ_ERR_INVALID, "null buffer");
  if (offset > b->size || bytes > b->size - offset) fail(NZ_ERR_INVALID, "copy exceeds buffer");
}
void copyDefault(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (stream) {
    NZ_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)));
  } else {
    NZ_CUDA(cudaMemcpy(dst, src, bytes, cudaMemcpyDefault));
  }
}
}  // namespace

int nz_buffer_write(nz_buf_t* b, uint64_t offset, const void* src, uint64_t bytes, void* stream) {
  return guarded([&] {
    copyChecked(b, offset, bytes);
    NZ_CUDA(cudaSetDevice(b->comm->device));
    if (bytes) copyDefault(b->ptrs[b->comm->rank] + offset, src, bytes, stream);
  });
}

int nz_buffer_read(const nz_buf_t* b, uint64_t offset, void* dst, uint64_t bytes, void* stream) {
  return guarded([&] {
    copyChecked(b, offset, bytes);
    NZ_CUDA(cudaSetDevice(b->comm->device));
    if (bytes) copyDefault(dst, b->ptrs[b->comm->rank] + offset, bytes, stream);
  });
}

int nz_buffer_fill_zero(nz_buf_t* b, void* stream) {
  return guarded([&] {
    if (!b) fail(NZ_ERR_INVALID, "null buffer");
    NZ_CUDA(cudaSetDevice(b->comm->device));
    if (stream) {
      NZ_CUDA(cudaMemsetAsync(b->ptrs[b->comm->rank], 0, b->size, static_cast<cudaStream_t>(stream)));
    } else {
      NZ_CUDA(cudaMemset(b->ptrs[b->comm->rank], 0, b->size));
    }
  });
}

}  // extern "C"
