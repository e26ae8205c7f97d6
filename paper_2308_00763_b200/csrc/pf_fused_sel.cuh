// Selection of the fused frame kernel's instantiations.  Each (precision,
// lane packing, debug) family is compiled in its own translation unit
// (pf_fused_inst.cu with -DPF_INST_M/PK/DBG, built in parallel by the
// Makefile); pf_api.cu launches them through these host-stub pointers.
#pragma once
#include "pf_kernels.cuh"

typedef void (*pf_fused_fn)(pfk::FusedArgs);

// (VPT, rounds) per threads-per-block: the tile is always PF_TILE particles
pf_fused_fn pf_fused_sel(int mode, bool pk, bool dbg, int tpb);
// sharded filters: 128 or 256 threads per block only (keeps the instantiations few)
pf_fused_fn pf_fused_sel_sharded(int mode, int tpb);
// numpy-philox stream: normals read from the generated buffer (128 / 256 threads)
pf_fused_fn pf_fused_sel_nz(int mode, bool pk, int tpb);
