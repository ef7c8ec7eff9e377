// fp_attn.cu -- stage (iii) dispatch (y = A(Q, K, V, S)):
// fp_attn8.cu (q-block pairs sharing K/V loads, ping-pong softmax warpgroups,
// persistent) for both block sizes: b = 128 directly, b = 64 (next
// row f3) as coarse 128 x 128 tiles with per-quadrant masks. Dense causal
// attention (the speedup denominator) does not depend on the block size.
#include "fp_internal.h"

namespace fp {

cudaError_t launch_attn_v8(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense, bool coarse,
                           int nb64, long long cap64, const void* const* peer_o, int n_peer, int* sched,
                           cudaStream_t st);

int attn_kv_box_rows() { return 128; }

cudaError_t launch_attn(const Shape& s, const WsLayout& L, void* ws, const Layout& lay,
                        const CUtensorMap& qmap, const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                        const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                        const void* const* peer_o, int n_peer, cudaStream_t st) {
  const Shape s128 = s.b == 128 ? s : make_shape(s.H, s.G, s.n, 128);
  const bool coarse = s.b != 128 && !dense;
  // persistent scheduler scratch (ws is optional: without it the kernel runs
  // one CTA per work item)
  int* sched = ws ? wsp<int>(ws, L.sched) : nullptr;
  return launch_attn_v8(s128, lay, qmap, kmap, vmap, o, row_ptr, col_idx, dense, coarse, s.nb, s.tri, peer_o,
                        n_peer, sched, st);
}

}  // namespace fp
