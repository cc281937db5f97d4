// ep_p2p.cu -- expert-parallel exchange over NVLink peer memory.
//
// With P2P (CUDA IPC-mapped) buffers the two collectives of an expert-parallel layer
// become loads and stores inside the kernels that produce / consume the data:
//   * dispatch: the router writes its ids/weights rows, and the previous layer's combine
//     writes the next token states h, straight into every rank's gathered buffers;
//   * combine: each rank's combine pass reads every slot's expert-output row from the
//     owner rank's y_perm (slot order and arithmetic of the single-GPU pass, so the step
//     stays bit-exact with one GPU).
// What remains is ordering: a one-warp flag barrier after the router (everybody's rows
// have landed) and after the FFN (everybody's y_perm is final). Flags live in each
// rank's peer-mapped memory; barrier i writes epoch i into slot `rank` of every rank's
// flag array (release, system scope) and waits until all of its own slots reach i
// (acquire). Epochs come from a device counter, so a CUDA graph of the step can be
// replayed. A barrier that waits longer than `timeout_ns` sets SERE_ERR_CUDA in the
// status word, raises the sticky abort word of every rank (params.cuh kEpAbortSlot) and
// returns instead of hanging the device.
#include <cuda_runtime.h>

#include "../../include/sere_b200.h"
#include "params.cuh"
#include "ptx.cuh"

namespace sere {

__global__ void __launch_bounds__(32) ep_barrier_kernel(const EpPeers ep, int32_t* epoch, int32_t* status,
                                                         long long timeout_ns) {
  __shared__ int s_epoch, s_abort;
  const int lane = threadIdx.x;
  if (lane == 0) {
    s_epoch = *epoch + 1;
    *epoch = s_epoch;
    s_abort = ep_aborted(ep);
  }
  __syncwarp();
  if (s_abort) {  // an earlier barrier of some rank timed out: fail fast, never wait
    if (lane == 0 && status) atomicExch(status, SERE_ERR_CUDA);
    return;
  }
  const int e = s_epoch;
  // the stream's earlier kernels (router / FFN) are complete; make their peer stores visible
  // system-wide before announcing the arrival
  __threadfence_system();
  if (lane < ep.world) st_release_sys(ep.flags[lane] + ep.rank, e);
  if (lane < ep.world) {
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(ep.flags[ep.rank] + lane) < e) {
      __nanosleep(100);
      if (globaltimer_ns() - t0 > static_cast<unsigned long long>(timeout_ns)) {
        if (status) atomicExch(status, SERE_ERR_CUDA);
        // sticky and visible to every rank: their next barrier fails fast and their peer
        // kernels skip the exchange (a late peer must not pass on this rank's newer epochs)
        for (int p = 0; p < ep.world; ++p) st_release_sys(ep.flags[p] + kEpAbortSlot, 1);
        break;
      }
    }
  }
  __syncwarp();
  __threadfence_system();
}

cudaError_t launch_ep_barrier(const EpPeers& ep, int32_t* epoch, int32_t* status, long long timeout_ns,
                              cudaStream_t stream) {
  ep_barrier_kernel<<<1, 32, 0, stream>>>(ep, epoch, status, timeout_ns);
  return cudaGetLastError();
}

}  // namespace sere
