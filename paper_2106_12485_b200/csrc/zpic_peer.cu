// zpic_peer.cu — the y-slab halo rounds written by the library's own kernels straight into the
// neighbours' receive areas (ZPIC_TRANSPORT_PEER / _LOOPBACK_PEER).
//
// Every context owns one "peer block" (cudaMalloc'd, so it can be exported with CUDA IPC): the
// raw J rows and the particle messages of round 1, the E/B ghost rows of round 2, and four epoch
// flags.  A neighbour's block is reached through a PeerView (its own pointers in a loopback
// group, CUDA IPC pointers across processes over NVLink, this context's own block in a one-rank
// ring).  A round is one copy kernel (the sender's rows and messages into the receiver's area, every
// thread ending with a system-scope fence), one signal kernel (a system-scope release store of the
// round's epoch into the receiver's flag) and, on the receiver, one wait kernel (an acquire spin
// until the flag reaches the epoch, bounded: a neighbour that never signals sets ERR_HALO instead
// of hanging the GPU).  Flags in the receiver's block: [0] round 1 from its lower neighbour, [1]
// round 1 from its upper one, [2] round 2 from the lower, [3] round 2 from the upper, [4] / [5] J
// zeroed by the lower / upper neighbour (cross-slab commutative current: from then on the
// neighbours' K1 may add into this slab's J).
// Reuse of an area is ordered by the protocol: a sender overwrites the receiver's round-1 area only
// after it waited for the receiver's round 2 of the previous step, which the receiver sends after it
// consumed that area.
#include <cuda_runtime.h>
#include <stdint.h>

#include "zpic_device.cuh"

namespace zpic {


// the peer block's layout (bytes), for a slab of row pitch `pitch` and message capacity pcap
struct PeerLayout {
  size_t jrup, jrdn, pmsg0, pmsg1, eb_lo, eb_hi, flags, bytes;
  PeerLayout(int pitch, int pcap) {
    const size_t rows2 = (size_t)3 * 2 * pitch * 4, mb = (msg_bytes(pcap) + 255) & ~(size_t)255;
    jrup = 0;
    jrdn = jrup + rows2;
    pmsg0 = jrdn + rows2;
    pmsg1 = pmsg0 + mb;
    eb_lo = pmsg1 + mb;
    eb_hi = eb_lo + (size_t)2 * 3 * pitch * 4;
    flags = eb_hi + (size_t)2 * 3 * 2 * pitch * 4;
    bytes = flags + 6 * sizeof(unsigned long long);
  }
};
PeerView peer_view(void* block, int pitch, int pcap) {
  const PeerLayout L(pitch, pcap);
  char* b = (char*)block;
  return PeerView{(float*)(b + L.jrup), (float*)(b + L.jrdn), {b + L.pmsg0, b + L.pmsg1}, (float*)(b + L.eb_lo),
                  (float*)(b + L.eb_hi), (unsigned long long*)(b + L.flags)};
}
size_t peer_block_bytes(int pitch, int pcap) { return PeerLayout(pitch, pcap).bytes; }

__device__ __forceinline__ const float* crow(const float* F, const GridDesc& g, int comp, int row) {
  return F + comp * g.plane + (long)(row + 1) * g.pitch;
}

// the first `count` records of a particle message (count in its header) into another message buffer
__device__ __forceinline__ void copy_msg(const char* src, char* dst, int pcap, long tid, long nthreads) {
  const PList S = msg_list(const_cast<char*>(src), pcap), D = msg_list(dst, pcap);
  const int n = min(*S.count, pcap);
  if (tid == 0) *D.count = n;
  for (long k = tid; k < 8L * n; k += nthreads) {
    const int f = (int)(k / n), q = (int)(k - (long)f * n);
    const uint32_t* s = f == 0 ? (const uint32_t*)S.cell : f == 1 ? (const uint32_t*)S.x : f == 2 ? (const uint32_t*)S.y
                      : f == 3 ? (const uint32_t*)S.ux : f == 4 ? (const uint32_t*)S.uy : f == 5 ? (const uint32_t*)S.uz
                      : f == 6 ? (const uint32_t*)S.id : (const uint32_t*)S.species;
    uint32_t* d = f == 0 ? (uint32_t*)D.cell : f == 1 ? (uint32_t*)D.x : f == 2 ? (uint32_t*)D.y : f == 3 ? (uint32_t*)D.ux
                : f == 4 ? (uint32_t*)D.uy : f == 5 ? (uint32_t*)D.uz : f == 6 ? (uint32_t*)D.id : (uint32_t*)D.species;
    d[q] = s[q];
  }
}

// Round 1: raw J rows ny, ny+1 and the up-going particles into the upper neighbour's area, raw J
// rows -1, 0 and the down-going particles into the lower neighbour's area (rows = 0: particles
// only; the cross-slab commutative current already added the rows into the neighbours' J).
__global__ void k_peer_put1(const float* J, GridDesc g, const char* send_dn, const char* send_up, int pcap,
                            PeerView lo, PeerView up, int has_lo, int has_hi, int rows) {
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long)gridDim.x * blockDim.x;
  const int P = g.pitch;
  for (long k = tid; k < (rows ? 6L * P : 0L); k += nth) {
    const int c = (int)(k / (2 * P)), r = (int)((k / P) % 2), x = (int)(k % P);
    if (has_hi) up.jrdn[(c * 2 + r) * P + x] = crow(J, g, c, g.ny + r)[x];
    if (has_lo) lo.jrup[(c * 2 + r) * P + x] = crow(J, g, c, r - 1)[x];
  }
  if (has_hi) copy_msg(send_up, up.pmsg[0], pcap, tid, nth);
  if (has_lo) copy_msg(send_dn, lo.pmsg[1], pcap, tid, nth);
  __threadfence_system();
}

// Round 2: E/B row ny-1 into the upper neighbour's guard-row area, rows 0, 1 into the lower's.
__global__ void k_peer_put2(const float* E, const float* B, GridDesc g, PeerView lo, PeerView up, int has_lo, int has_hi) {
  const long tid = (long)blockIdx.x * blockDim.x + threadIdx.x, nth = (long)gridDim.x * blockDim.x;
  const int P = g.pitch;
  for (long k = tid; k < 6L * P; k += nth) {   // (field, comp) pairs x pitch
    const int fc = (int)(k / P), x = (int)(k % P), f = fc / 3, c = fc % 3;
    const float* F = f ? B : E;
    if (has_hi) up.eb_lo[fc * P + x] = crow(F, g, c, g.ny - 1)[x];
    if (has_lo) {
      lo.eb_hi[(fc * 2 + 0) * P + x] = crow(F, g, c, 0)[x];
      lo.eb_hi[(fc * 2 + 1) * P + x] = crow(F, g, c, 1)[x];
    }
  }
  __threadfence_system();
}

// The receiver's guard rows from its round-2 area.
__global__ void k_peer_apply2(float* E, float* B, GridDesc g, const float* eb_lo, const float* eb_hi, int has_lo,
                              int has_hi) {
  const int P = g.pitch;
  for (long k = (long)blockIdx.x * blockDim.x + threadIdx.x; k < 6L * P; k += (long)gridDim.x * blockDim.x) {
    const int fc = (int)(k / P), x = (int)(k % P), f = fc / 3, c = fc % 3;
    float* F = f ? B : E;
    if (has_lo) F[c * g.plane + (long)(-1 + 1) * P + x] = eb_lo[fc * P + x];
    if (has_hi) {
      F[c * g.plane + (long)(g.ny + 1) * P + x] = eb_hi[(fc * 2 + 0) * P + x];
      F[c * g.plane + (long)(g.ny + 2) * P + x] = eb_hi[(fc * 2 + 1) * P + x];
    }
  }
}

// One thread: release-store the epoch into up to two receivers' flags (system scope: NVLink peers).
__global__ void k_peer_signal(unsigned long long* fa, unsigned long long* fb, unsigned long long e) {
  if (fa) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fa), "l"(e) : "memory");
  if (fb) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(fb), "l"(e) : "memory");
}

// One thread: acquire-spin until flags[ia] (and flags[ib]) reach the epoch (-1: not waited for).
// A wait is always enqueued after the signal it reads when both ranks share a stream (loopback
// groups, the one-rank ring), so on one GPU no wait kernel depends on a concurrently running one.
// Bounded (~20 s of GPU clock): a neighbour that never signals sets ERR_HALO instead of hanging.
__global__ void k_peer_wait(const unsigned long long* flags, int ia, int ib, unsigned long long e, int* err) {
  const long long t0 = clock64();
  for (int q = 0; q < 2; ++q) {
    const int i = q ? ib : ia;
    if (i < 0) continue;
    unsigned long long v;
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + i) : "memory");
      if (v >= e) break;
      if (clock64() - t0 > 40000000000LL) { atomicOr(err, ERR_HALO); return; }
      __nanosleep(256);
    }
  }
}

void launch_peer_put1(const float* J, const GridDesc& g, const void* send_dn, const void* send_up, int pcap,
                      const PeerView& lo, const PeerView& up, int has_lo, int has_hi, int rows, cudaStream_t st) {
  k_peer_put1<<<148, 256, 0, st>>>(J, g, (const char*)send_dn, (const char*)send_up, pcap, lo, up, has_lo, has_hi,
                                   rows);
}
void launch_peer_put2(const float* E, const float* B, const GridDesc& g, const PeerView& lo, const PeerView& up,
                      int has_lo, int has_hi, cudaStream_t st) {
  k_peer_put2<<<148, 256, 0, st>>>(E, B, g, lo, up, has_lo, has_hi);
}
void launch_peer_apply2(float* E, float* B, const GridDesc& g, const PeerView& self, int has_lo, int has_hi,
                        cudaStream_t st) {
  k_peer_apply2<<<148, 256, 0, st>>>(E, B, g, self.eb_lo, self.eb_hi, has_lo, has_hi);
}
void launch_peer_signal(unsigned long long* fa, unsigned long long* fb, unsigned long long e, cudaStream_t st) {
  k_peer_signal<<<1, 1, 0, st>>>(fa, fb, e);
}
void launch_peer_wait(const unsigned long long* flags, int ia, int ib, unsigned long long e, int* err, cudaStream_t st) {
  k_peer_wait<<<1, 1, 0, st>>>(flags, ia, ib, e, err);
}

}  // namespace zpic
