// zpic_peer.cu — the y-slab halo rounds written by the library's own kernels straight into the
// neighbours' receive areas (ZPIC_TRANSPORT_PEER / _LOOPBACK_PEER).
//
// Every context owns one "peer block" (cudaMalloc'd, so it can be exported with CUDA IPC): the
// raw J rows and the particle messages of round 1, the E/B ghost rows of round 2, and six epoch
// flags.  A neighbour's block is reached through a PeerView (its own pointers in a loopback
// group, CUDA IPC pointers across processes over NVLink, this context's own block in a one-rank
// ring).  The particles leaving the slab are appended straight into the neighbour's message area
// by the kernels that route them (K3, K1L: a slot from the receiver's count, then the record; the
// receiver zeroes its counts once it inserted them), and the E/B rows of round 2 by K5's slab-edge
// tiles straight into the neighbours' guard rows (k_peer_put2 below only after zpic_set_fields).
// A round is then at most one copy kernel (the sender's raw J rows into the receiver's area; none
// with the cross-slab commutative current), every writer ending with a system-scope fence, one signal kernel (a
// system-scope release store of the round's epoch into the receiver's flag) and, on the receiver,
// one wait kernel (an acquire spin until the flag reaches the epoch, bounded: a neighbour that
// never signals sets ERR_HALO instead of hanging the GPU).  Flags in the receiver's block: [0] round 1 from its lower neighbour, [1]
// round 1 from its upper one, [2] round 2 from the lower, [3] round 2 from the upper, [4] / [5] J
// zeroed by the lower / upper neighbour (cross-slab commutative current: from then on the
// neighbours' K1 may add into this slab's J).
// Reuse of an area is ordered by the protocol: a sender writes the receiver's round-1 area (J rows,
// message records) only after it waited for the receiver's round 2 of the previous step, which the
// receiver sends after it consumed that area (and zeroed its message counts); the slab exits are
// appended by K3 / K1L, which run after that wait (the next step's boundary K1).
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "zpic_device.cuh"

namespace zpic {


// the peer block's layout (bytes), for a slab of row pitch `pitch` and message capacity pcap
struct PeerLayout {
  size_t jrup, jrdn, pmsg0, pmsg1, flags, bytes;
  PeerLayout(int pitch, int pcap) {
    const size_t rows2 = (size_t)3 * 2 * pitch * 4, mb = (msg_bytes(pcap) + 255) & ~(size_t)255;
    jrup = 0;
    jrdn = jrup + rows2;
    pmsg0 = jrdn + rows2;
    pmsg1 = pmsg0 + mb;
    flags = pmsg1 + mb;
    bytes = flags + 6 * sizeof(unsigned long long);
  }
};
PeerView peer_view(void* block, int pitch, int pcap) {
  const PeerLayout L(pitch, pcap);
  char* b = (char*)block;
  PeerView v{};
  v.jrup = (float*)(b + L.jrup);
  v.jrdn = (float*)(b + L.jrdn);
  v.pmsg[0] = b + L.pmsg0;
  v.pmsg[1] = b + L.pmsg1;
  v.flags = (unsigned long long*)(b + L.flags);
  return v;   // E, B, plane, ny: set by the owner (field buffers)
}
size_t peer_block_bytes(int pitch, int pcap) { return PeerLayout(pitch, pcap).bytes; }

__device__ __forceinline__ const float* crow(const float* F, const GridDesc& g, int comp, int row) {
  return F + comp * g.plane + (long)(row + 1) * g.pitch;
}

// Round 1: raw J rows ny, ny+1 into the upper neighbour's area, raw J rows -1, 0 into the lower
// neighbour's.  The particles leaving the slab need no copy: K3 and K1L append them straight into
// the neighbours' message areas (PushParams.send, peer_send).  With the cross-slab commutative
// current there is nothing to put (K1 / K1L added the rows into the neighbours' J).  Thread tid of
// nth; the caller fences (system scope) before the round is signalled.
__device__ __forceinline__ void put1_body(const float* J, const GridDesc& g, const PeerView& lo, const PeerView& up,
                                          int has_lo, int has_hi, long tid, long nth) {
  const int P = g.pitch;
  for (long k = tid; k < 6L * P; k += nth) {
    const int c = (int)(k / (2 * P)), r = (int)((k / P) % 2), x = (int)(k % P);
    if (has_hi) up.jrdn[(c * 2 + r) * P + x] = crow(J, g, c, g.ny + r)[x];
    if (has_lo) lo.jrup[(c * 2 + r) * P + x] = crow(J, g, c, r - 1)[x];
  }
}
__global__ void k_peer_put1(const float* J, GridDesc g, PeerView lo, PeerView up, int has_lo, int has_hi) {
  put1_body(J, g, lo, up, has_lo, has_hi, (long)blockIdx.x * blockDim.x + threadIdx.x, (long)gridDim.x * blockDim.x);
  __threadfence_system();
}

// Round 2: E/B row ny-1 (buffer b) into the upper neighbour's guard row -1, rows 0, 1 into the
// lower neighbour's guard rows ny, ny + 1 — straight into their field buffers of the same parity
// (no receive area, no apply pass: the slab-edge CTAs of the next K1 wait for the flag and read
// them with their TMA field boxes).
__device__ __forceinline__ void put2_body(const float* E, const float* B, const GridDesc& g, const PeerView& lo,
                                          const PeerView& up, int has_lo, int has_hi, int b, long tid, long nth) {
  const int P = g.pitch;
  for (long k = tid; k < 6L * P; k += nth) {   // (field, comp) pairs x pitch
    const int fc = (int)(k / P), x = (int)(k % P), f = fc / 3, c = fc % 3;
    const float* F = f ? B : E;
    if (has_hi) (f ? up.B[b] : up.E[b])[c * up.plane + x] = crow(F, g, c, g.ny - 1)[x];
    if (has_lo) {
      float* D = (f ? lo.B[b] : lo.E[b]) + c * lo.plane + (long)(lo.ny + 1) * P + x;
      D[0] = crow(F, g, c, 0)[x];
      D[P] = crow(F, g, c, 1)[x];
    }
  }
}
__global__ void k_peer_put2(const float* E, const float* B, GridDesc g, PeerView lo, PeerView up, int has_lo, int has_hi,
                            int b) {
  put2_body(E, B, g, lo, up, has_lo, has_hi, b, (long)blockIdx.x * blockDim.x + threadIdx.x,
            (long)gridDim.x * blockDim.x);
  __threadfence_system();
}

// One thread: release-store the epoch into up to two receivers' flags.
__global__ void k_peer_signal(unsigned long long* fa, unsigned long long* fb, unsigned long long e) {
  if (fa) signal_flag(fa, e);
  if (fb) signal_flag(fb, e);
}

// One thread: wait for the round's flags.  Bounded (~20 s of GPU clock): a neighbour that never
// signals sets ERR_HALO instead of hanging.
// A wait is always enqueued after the signal it reads when both ranks share a stream (loopback
// groups, the one-rank ring), so on one GPU no wait kernel depends on a concurrently running one.
__global__ void k_peer_wait(const unsigned long long* flags, int ia, int ib, unsigned long long e, int* err) {
  if (!wait_flags(flags, ia, ib, e, 40000000000LL)) atomicOr(err, ERR_HALO);
}

void launch_peer_put1(const float* J, const GridDesc& g, const PeerView& lo, const PeerView& up, int has_lo,
                      int has_hi, cudaStream_t st) {
  k_peer_put1<<<48, 256, 0, st>>>(J, g, lo, up, has_lo, has_hi);
}
void launch_peer_put2(const float* E, const float* B, const GridDesc& g, const PeerView& lo, const PeerView& up,
                      int has_lo, int has_hi, int b, cudaStream_t st) {
  k_peer_put2<<<48, 256, 0, st>>>(E, B, g, lo, up, has_lo, has_hi, b);
}
void launch_peer_signal(unsigned long long* fa, unsigned long long* fb, unsigned long long e, cudaStream_t st) {
  k_peer_signal<<<1, 1, 0, st>>>(fa, fb, e);
}
void launch_peer_wait(const unsigned long long* flags, int ia, int ib, unsigned long long e, int* err, cudaStream_t st) {
  k_peer_wait<<<1, 1, 0, st>>>(flags, ia, ib, e, err);
}

// ---- protocol self-test (zpic_peer_selftest) -------------------------------------------------
// `ranks` emulated slabs of a ring (or chain), one CTA each, in ONE cooperative launch (all CTAs
// co-resident), run `epochs` steps of the PEER protocol with the production bodies above: round 1
// (put1_body: J rows + particle messages into the neighbours' areas), signal, wait, consume (here:
// verify against the content the neighbour wrote for this epoch), round 2 (put2_body), signal,
// wait, verify.  The waits really spin on flags other CTAs store concurrently, which the loopback
// groups (one stream, every signal before its wait) never do, so this checks the flag indices, the
// epochs and the reuse of the receive areas under true concurrency on one GPU (the profiling
// guide's rule: emulate the ranks inside one kernel rather than as ranks that wait on one another).
struct SelfRank {
  float* J;
  float* E;
  float* B;
  PeerView self, lo, hi;
  int has_lo, has_hi, lower, upper;
  float* Jn[2];              // the lower / upper neighbour's J (commutative mode)
  long lo_plane, hi_plane;
  int lo_ny;
};
__device__ __forceinline__ uint32_t st_hash(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA77u ^ (c + 0x165667B1u) * 0xC2B2AE3Du ^ d * 0x27D4EB2Fu;
  h ^= h >> 15; h *= 0x2C1B3C6Du; h ^= h >> 12;
  return h;
}
__device__ __forceinline__ float st_val(uint32_t h) { return (float)(h & 0xFFFFF); }   // exact in fp32
// what rank r writes, at epoch e, into row `row` (-1 .. ny+1) of component c of J / E / B
__device__ __forceinline__ float st_row(int r, int e, int what, int c, int row, int x) {
  return st_val(st_hash(r, e, what * 8 + c, (uint32_t)(row + 2) * 65536u + x));
}
__device__ __forceinline__ int st_count(int r, int e, int d, int pcap) { return (int)(st_hash(r, e, 99, d) % (pcap + 1)); }

// fault (checks that the self-test can fail): 1 = rank 0 overwrites one value of its round-1 J rows in
// the upper neighbour's area at epoch 2 after the put (a wrong value the receiver must see);
// 2 = rank 0 does not signal round 1 at epoch 2 (its neighbours' waits must time out).
// commutative = 1: the cross-slab commutative current instead of J rows in round 1: every epoch
// each rank zeroes its J, signals "zeroed" (flags 4 / 5), waits for its neighbours' "zeroed", adds
// its contributions on rows -1, 0, ny, ny + 1 into its own J and through peer_add_j into the
// neighbours' J (RED over peer memory), fences, and round 1 then carries the particles only; after
// the round-1 wait the shared rows must hold own + neighbour contribution exactly (small integers).
__global__ void k_peer_selftest(SelfRank* ranks, GridDesc g, int pcap, int epochs, long long budget, int fault,
                                int commutative, unsigned long long* errors) {
  const SelfRank me = ranks[blockIdx.x];
  const int r = blockIdx.x, tid = threadIdx.x, nth = blockDim.x, P = g.pitch;
  __shared__ int s_ok;
  __shared__ unsigned s_seen[4096 / 32];   // records received this epoch (pcap <= 4096)
  unsigned long long bad = 0;
  for (int e = 1; e <= epochs; ++e) {
    if (commutative) {
      for (long k = tid; k < 3 * g.plane; k += nth) me.J[k] = 0.f;
      __threadfence_system();
      __syncthreads();
      if (tid == 0) {
        if (me.has_hi) signal_flag(me.hi.flags + 4, e);
        if (me.has_lo) signal_flag(me.lo.flags + 5, e);
        s_ok = wait_flags(me.self.flags, me.has_lo ? 4 : -1, me.has_hi ? 5 : -1, e, budget);
        __threadfence();
      }
      __syncthreads();
      if (!s_ok) { if (tid == 0) atomicAdd(errors, 1ull << 40); return; }
      float* Jlo = me.has_lo ? me.Jn[0] : nullptr;
      float* Jhi = me.has_hi ? me.Jn[1] : nullptr;
      for (int k = tid; k < 3 * 4 * P; k += nth) {
        const int c = k / (4 * P), q = (k / P) % 4, x = k % P, row = q < 2 ? q - 1 : g.ny + q - 2;
        const long o = (long)(row + 1) * P + x;
        const float v = st_row(r, e, 0, c, row, x);
        atomicAdd(me.J + c * g.plane + o, v);
        peer_add_j(Jlo, Jhi, me.lo_plane, me.hi_plane, me.lo_ny, g, c, row, o, v);
      }
    } else {
      // this rank's J rows and messages of epoch e (its own buffers)
      for (int k = tid; k < 3 * 4 * P; k += nth) {
        const int c = k / (4 * P), q = (k / P) % 4, x = k % P, row = q < 2 ? q - 1 : g.ny + q - 2;
        me.J[c * g.plane + (long)(row + 1) * P + x] = st_row(r, e, 0, c, row, x);
      }
    }
    // this epoch's slab exits, appended straight into the neighbours' message areas as K3 / K1L do
    // (list_append: a slot from the receiver's count, then the record); record k carries id = k
    for (int d = 0; d < 2; ++d) {
      if (d == 0 ? !me.has_lo : !me.has_hi) continue;
      const PList L = msg_list(d == 0 ? me.lo.pmsg[1] : me.hi.pmsg[0], pcap);
      const int n = st_count(r, e, d, pcap);
      for (int k = tid; k < n; k += nth) {
        const uint32_t h = st_hash(r, e, 100 + d, k);
        list_append(L, reinterpret_cast<int*>(errors), (int)h, st_val(h ^ 1), st_val(h ^ 2), st_val(h ^ 3),
                    st_val(h ^ 4), st_val(h ^ 5), (uint32_t)k, (int)(h & 3));
      }
    }
    __syncthreads();
    if (!commutative) put1_body(me.J, g, me.lo, me.hi, me.has_lo, me.has_hi, tid, nth);
    if (fault == 1 && r == 0 && e == 2 && tid == 0 && me.has_hi) {
      if (commutative) atomicAdd(me.Jn[1] + P + 3, 1.0f);   // (upper's row 0, column -1)
      else me.hi.jrdn[P + 3] += 1.0f;
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
      const bool drop = fault == 2 && r == 0 && e == 2;
      if (me.has_hi && !drop) signal_flag(me.hi.flags + 0, e);
      if (me.has_lo && !drop) signal_flag(me.lo.flags + 1, e);
      s_ok = wait_flags(me.self.flags, me.has_lo ? 0 : -1, me.has_hi ? 1 : -1, e, budget);
      __threadfence();
    }
    __syncthreads();
    if (!s_ok) { if (tid == 0) atomicAdd(errors, 1ull << 40); return; }
    // consume round 1: the lower's raw rows ny, ny+1 and up-going particles, the upper's rows -1, 0
    // and down-going particles
    for (int k = tid; k < 6 * P; k += nth) {
      const int c = k / (2 * P), q = (k / P) % 2, x = k % P;
      if (commutative) {   // rows 0, 1 = own + the lower's rows ny, ny + 1; rows ny - 1, ny = own + the upper's -1, 0
        const float* Jc = me.J + c * g.plane;
        const float lo0 = st_row(r, e, 0, c, q, x) * (q == 0 ? 1.f : 0.f);   // own deposits only on rows 0 (not 1)
        const float hi0 = st_row(r, e, 0, c, g.ny - 1 + q, x) * (q == 1 ? 1.f : 0.f);   // own only on row ny
        if (me.has_lo && Jc[(long)(q + 1) * P + x] != lo0 + st_row(me.lower, e, 0, c, g.ny + q, x)) ++bad;
        if (me.has_hi && Jc[(long)(g.ny + q) * P + x] != hi0 + st_row(me.upper, e, 0, c, q - 1, x)) ++bad;
      } else {
        if (me.has_lo && me.self.jrdn[(c * 2 + q) * P + x] != st_row(me.lower, e, 0, c, g.ny + q, x)) ++bad;
        if (me.has_hi && me.self.jrup[(c * 2 + q) * P + x] != st_row(me.upper, e, 0, c, q - 1, x)) ++bad;
      }
    }
    for (int side = 0; side < 2; ++side) {   // pmsg[0] from the lower (its up messages), [1] from the upper
      if (side == 0 ? !me.has_lo : !me.has_hi) continue;
      const int from = side == 0 ? me.lower : me.upper, d = side == 0 ? 1 : 0;
      const PList L = msg_list(me.self.pmsg[side], pcap);
      const int n = st_count(from, e, d, pcap);
      for (int k = tid; k < 4096 / 32; k += nth) s_seen[k] = 0u;
      __syncthreads();
      if (tid == 0 && *L.count != n) ++bad;
      for (int q = tid; q < min(*L.count, pcap); q += nth) {   // any order; every record k < n exactly once
        const uint32_t k = L.id[q];
        const uint32_t h = st_hash(from, e, 100 + d, k);
        if (k >= (uint32_t)n || L.cell[q] != (int)h || L.x[q] != st_val(h ^ 1) || L.y[q] != st_val(h ^ 2) ||
            L.ux[q] != st_val(h ^ 3) || L.uy[q] != st_val(h ^ 4) || L.uz[q] != st_val(h ^ 5) ||
            L.species[q] != (int)(h & 3) || (atomicOr(&s_seen[k >> 5], 1u << (k & 31)) >> (k & 31)) & 1u)
          ++bad;
      }
      __syncthreads();
      if (tid == 0) *L.count = 0;   // consumed (as after k_recv_insert): the sender appends from zero
    }
    // round 2: this rank's E / B rows 0, 1, ny - 1 of epoch e
    for (int k = tid; k < 2 * 3 * 3 * P; k += nth) {
      const int f = k / (9 * P), c = (k / (3 * P)) % 3, q = (k / P) % 3, x = k % P, row = q < 2 ? q : g.ny - 1;
      (f ? me.B : me.E)[c * g.plane + (long)(row + 1) * P + x] = st_row(r, e, 1 + f, c, row, x);
    }
    __syncthreads();
    put2_body(me.E, me.B, g, me.lo, me.hi, me.has_lo, me.has_hi, 0, tid, nth);
    __threadfence_system();
    __syncthreads();
    if (tid == 0) {
      if (me.has_hi) signal_flag(me.hi.flags + 2, e);
      if (me.has_lo) signal_flag(me.lo.flags + 3, e);
      s_ok = wait_flags(me.self.flags, me.has_lo ? 2 : -1, me.has_hi ? 3 : -1, e, budget);
      __threadfence();
    }
    __syncthreads();
    if (!s_ok) { if (tid == 0) atomicAdd(errors, 1ull << 40); return; }
    for (int k = tid; k < 6 * P; k += nth) {   // (field, comp) x pitch
      const int fc = k / P, x = k % P, f = fc / 3, c = fc % 3;
      const float* F = (f ? me.B : me.E) + c * g.plane;   // this rank's guard rows -1, ny, ny + 1
      if (me.has_lo && F[x] != st_row(me.lower, e, 1 + f, c, g.ny - 1, x)) ++bad;
      if (me.has_hi && (F[(long)(g.ny + 1) * P + x] != st_row(me.upper, e, 1 + f, c, 0, x) ||
                        F[(long)(g.ny + 2) * P + x] != st_row(me.upper, e, 1 + f, c, 1, x)))
        ++bad;
    }
    __syncthreads();   // every thread verified this epoch's areas before the next epoch's round 1
  }
  if (bad) atomicAdd(errors, bad);
}

}  // namespace zpic

using namespace zpic;

extern "C" zpic_status zpic_peer_selftest(int32_t ranks, int32_t epochs, int32_t nx, int32_t ny, int32_t pcap,
                                          int32_t periodic, int32_t commutative, int64_t budget_cycles, int32_t fault,
                                          int64_t* errors_out) {
  if (ranks < 1 || ranks > 64 || epochs < 1 || nx < 1 || ny < 4 || pcap < 32 || pcap > 4096 || !errors_out)
    return ZPIC_E_INVALID;
  GridDesc g;
  g.nx = nx; g.ny = ny;
  g.pitch = (nx + kXOff + 2 + 31) / 32 * 32;
  g.rows = ny + 3;
  g.plane = (long)g.rows * g.pitch;
  std::vector<void*> mem;
  auto dalloc = [&](size_t b) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, b) != cudaSuccess) return nullptr;
    mem.push_back(p);
    cudaMemset(p, 0, b);
    return p;
  };
  zpic_status st = ZPIC_OK;
  std::vector<SelfRank> hr(ranks);
  std::vector<PeerView> views(ranks);
  for (int r = 0; r < ranks && st == ZPIC_OK; ++r) {
    void* blk = dalloc(peer_block_bytes(g.pitch, pcap));
    float* J = (float*)dalloc(3 * g.plane * sizeof(float));
    float* E = (float*)dalloc(3 * g.plane * sizeof(float));
    float* B = (float*)dalloc(3 * g.plane * sizeof(float));
    if (!blk || !J || !E || !B) { st = ZPIC_E_CUDA; break; }
    views[r] = peer_view(blk, g.pitch, pcap);
    views[r].E[0] = views[r].E[1] = E;
    views[r].B[0] = views[r].B[1] = B;
    views[r].plane = g.plane;
    views[r].ny = g.ny;
    hr[r].J = J; hr[r].E = E; hr[r].B = B;
  }
  if (st == ZPIC_OK) {
    for (int r = 0; r < ranks; ++r) {
      hr[r].lower = (r + ranks - 1) % ranks;
      hr[r].upper = (r + 1) % ranks;
      hr[r].has_lo = periodic || r > 0;
      hr[r].has_hi = periodic || r < ranks - 1;
      hr[r].self = views[r];
      hr[r].lo = views[hr[r].lower];
      hr[r].hi = views[hr[r].upper];
      hr[r].Jn[0] = hr[hr[r].lower].J;
      hr[r].Jn[1] = hr[hr[r].upper].J;
      hr[r].lo_plane = hr[r].hi_plane = g.plane;
      hr[r].lo_ny = g.ny;
    }
    SelfRank* dr = (SelfRank*)dalloc(sizeof(SelfRank) * ranks);
    unsigned long long* derr = (unsigned long long*)dalloc(sizeof(unsigned long long));
    if (!dr || !derr) st = ZPIC_E_CUDA;
    if (st == ZPIC_OK) {
      cudaMemcpy(dr, hr.data(), sizeof(SelfRank) * ranks, cudaMemcpyHostToDevice);
      long long budget = budget_cycles;
      int pc = pcap, ep = epochs, fl = fault, cm = commutative;
      void* args[] = {&dr, &g, &pc, &ep, &budget, &fl, &cm, &derr};
      if (cudaLaunchCooperativeKernel((const void*)k_peer_selftest, dim3(ranks), dim3(256), args, 0, 0) != cudaSuccess ||
          cudaDeviceSynchronize() != cudaSuccess) {
        st = ZPIC_E_CUDA;
      } else {
        unsigned long long h = 0;
        cudaMemcpy(&h, derr, sizeof(h), cudaMemcpyDeviceToHost);
        *errors_out = (int64_t)h;
      }
    }
  }
  for (void* p : mem) cudaFree(p);
  return st;
}
