// fp_attn.cu -- stage (iii) dispatch (y = A(Q, K, V, S)):
// block size 128 runs fp_attn8.cu (q-block pairs sharing K/V loads, ping-pong
// softmax warpgroups); block size 64 (next row f3) runs
// fp_attn64.cu. Dense causal attention (the speedup denominator) does not
// depend on the block size and always uses the 128 kernel.
#include "fp_internal.h"

namespace fp {

cudaError_t launch_attn_v8(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                           const void* const* peer_o, int n_peer, int* sched, cudaStream_t st);
cudaError_t launch_attn_b64(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                            const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                            const int32_t* row_ptr, const int32_t* col_idx, cudaStream_t st);

int attn_kv_box_rows() { return 128; }

cudaError_t launch_attn(const Shape& s, const WsLayout& L, void* ws, const Layout& lay,
                        const CUtensorMap& qmap, const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                        const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                        const void* const* peer_o, int n_peer, cudaStream_t st) {
  if (s.b != 128 && !dense) {
    if (n_peer > 0) return cudaErrorNotSupported;  // the fused output exchange is v8's
    return launch_attn_b64(s, lay, qmap, kmap, vmap, o, row_ptr, col_idx, st);
  }
  const Shape s128 = s.b == 128 ? s : make_shape(s.H, s.G, s.n, 128);
  // persistent scheduler scratch (ws is optional: without it the exact kernel
  // runs one CTA per work item)
  int* sched = ws ? wsp<int>(ws, L.sched) : nullptr;
  return launch_attn_v8(s128, lay, qmap, kmap, vmap, o, row_ptr, col_idx, dense, peer_o, n_peer, sched, st);
}

}  // namespace fp
