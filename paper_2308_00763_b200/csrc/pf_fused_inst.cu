// One family of pf_fused_frame instantiations per translation unit (see
// pf_fused_sel.cuh): PF_INST_M (0 FP64, 1 FP32, 2 FP16), PF_INST_PK (half2
// lanes), PF_INST_DBG (trace / debug-capture variant).  The unit with
// PF_INST_SEL defines the selection functions over all families.
#define PF_FUSED_ONLY
#include "pf_fused_sel.cuh"

#ifndef PF_INST_SEL
#define PF_FAMILY_FN(M, PK, DBG) pf_fused_family_##M##_##PK##_##DBG
#define PF_FAMILY(M, PK, DBG) PF_FAMILY_FN(M, PK, DBG)
// unsharded, LCG stream, every block size
pf_fused_fn PF_FAMILY(PF_INST_M, PF_INST_PK, PF_INST_DBG)(int tpb) {
  constexpr int M = PF_INST_M;
  constexpr bool PK = PF_INST_PK, DBG = PF_INST_DBG;
  switch (tpb) {
    case 32: return pfk::pf_fused_frame<M, 8, 4, false, PK, DBG>;
    case 64: return pfk::pf_fused_frame<M, 8, 2, false, PK, DBG>;
    case 128: return pfk::pf_fused_frame<M, 8, 1, false, PK, DBG>;
    case 512: return pfk::pf_fused_frame<M, 2, 1, false, PK, DBG>;
    case 1024: return pfk::pf_fused_frame<M, 1, 1, false, PK, DBG>;
    default: return pfk::pf_fused_frame<M, 4, 1, false, PK, DBG>;
  }
}
#if !PF_INST_DBG
// the production families also carry the sharded (packed lanes) and
// numpy-philox variants of their precision
#if PF_INST_PK
pf_fused_fn PF_FAMILY(PF_INST_M, sh, 0)(int tpb) {
  constexpr int M = PF_INST_M;
  return tpb == 128 ? pfk::pf_fused_frame<M, 8, 1, true> : pfk::pf_fused_frame<M, 4, 1, true>;
}
#endif
pf_fused_fn PF_FAMILY(PF_INST_M, nz, PF_INST_PK)(int tpb) {
  constexpr int M = PF_INST_M;
  constexpr bool PK = PF_INST_PK;
  return tpb == 128 ? pfk::pf_fused_frame<M, 8, 1, false, PK, false, true>
                    : pfk::pf_fused_frame<M, 4, 1, false, PK, false, true>;
}
#endif
#else
#define DECL(M, PK, DBG) pf_fused_fn pf_fused_family_##M##_##PK##_##DBG(int tpb);
DECL(0, 1, 0) DECL(0, 1, 1) DECL(1, 1, 0) DECL(1, 1, 1) DECL(2, 1, 0) DECL(2, 1, 1) DECL(2, 0, 0) DECL(2, 0, 1)
DECL(0, sh, 0) DECL(1, sh, 0) DECL(2, sh, 0) DECL(0, nz, 1) DECL(1, nz, 1) DECL(2, nz, 1) DECL(2, nz, 0)
#undef DECL

pf_fused_fn pf_fused_sel(int mode, bool pk, bool dbg, int tpb) {
  if (mode == 0) return dbg ? pf_fused_family_0_1_1(tpb) : pf_fused_family_0_1_0(tpb);
  if (mode == 1) return dbg ? pf_fused_family_1_1_1(tpb) : pf_fused_family_1_1_0(tpb);
  if (pk) return dbg ? pf_fused_family_2_1_1(tpb) : pf_fused_family_2_1_0(tpb);
  return dbg ? pf_fused_family_2_0_1(tpb) : pf_fused_family_2_0_0(tpb);
}
pf_fused_fn pf_fused_sel_sharded(int mode, int tpb) {
  return mode == 0 ? pf_fused_family_0_sh_0(tpb) : mode == 1 ? pf_fused_family_1_sh_0(tpb) : pf_fused_family_2_sh_0(tpb);
}
pf_fused_fn pf_fused_sel_nz(int mode, bool pk, int tpb) {
  if (mode == 0) return pf_fused_family_0_nz_1(tpb);
  if (mode == 1) return pf_fused_family_1_nz_1(tpb);
  return pk ? pf_fused_family_2_nz_1(tpb) : pf_fused_family_2_nz_0(tpb);
}
#endif
