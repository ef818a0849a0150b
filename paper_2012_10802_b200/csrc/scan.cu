// scan.cu — workspace of the single-pass scan (scan.cuh).
#include "scan.cuh"

namespace rpdg {

ScanState scan_state(rpd_ctx* ctx, long long n) {
  if (n >= (1ll << 30)) throw InvalidArg("scan: more than 2^30 elements");
  const long long tiles = (n + scan_detail::kScanTile - 1) / scan_detail::kScanTile;
  auto* desc = ctx->ws.get<unsigned long long>("scan_desc", size_t(tiles));
  auto* ctl = ctx->ws.get<unsigned>("scan_ctl", 2);
  // descriptors are tagged per launch: zero once per allocation (tag 0 never
  // matches a launch's tag), the control words likewise
  if (ctx->scan_zeroed != desc || ctx->scan_zeroed_tiles < tiles) {
    RPD_CK(cudaMemsetAsync(desc, 0, sizeof(unsigned long long) * size_t(tiles), ctx->stream));
    ctx->scan_zeroed = desc;
    ctx->scan_zeroed_tiles = tiles;
  }
  if (ctx->scan_ctl_zeroed != ctl) {
    RPD_CK(cudaMemsetAsync(ctl, 0, 2 * sizeof(unsigned), ctx->stream));
    ctx->scan_ctl_zeroed = ctl;
  }
  return ScanState{desc, ctl, unsigned(tiles)};
}

void scan_exclusive_i32(rpd_ctx* ctx, const int* in, int* out, long long n) {
  scan_exclusive(ctx, ScanArrayIn{in}, out, n);
}

}  // namespace rpdg
