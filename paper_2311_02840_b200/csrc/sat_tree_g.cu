// sat_tree_g.cu -- explicit instantiations of launch_tree_g<G> for G in [SAT_G_LO, SAT_G_HI];
// compiled several times with different ranges so the 32 specialisations build in parallel.
#include "sat_tree.cuh"

#ifndef SAT_G_LO
#define SAT_G_LO 1
#define SAT_G_HI 32
#endif

namespace sat {
#if SAT_G_LO <= 1 && 1 <= SAT_G_HI
template int launch_tree_g<1>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 2 && 2 <= SAT_G_HI
template int launch_tree_g<2>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 3 && 3 <= SAT_G_HI
template int launch_tree_g<3>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 4 && 4 <= SAT_G_HI
template int launch_tree_g<4>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 5 && 5 <= SAT_G_HI
template int launch_tree_g<5>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 6 && 6 <= SAT_G_HI
template int launch_tree_g<6>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 7 && 7 <= SAT_G_HI
template int launch_tree_g<7>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 8 && 8 <= SAT_G_HI
template int launch_tree_g<8>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 9 && 9 <= SAT_G_HI
template int launch_tree_g<9>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 10 && 10 <= SAT_G_HI
template int launch_tree_g<10>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 11 && 11 <= SAT_G_HI
template int launch_tree_g<11>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 12 && 12 <= SAT_G_HI
template int launch_tree_g<12>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 13 && 13 <= SAT_G_HI
template int launch_tree_g<13>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 14 && 14 <= SAT_G_HI
template int launch_tree_g<14>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 15 && 15 <= SAT_G_HI
template int launch_tree_g<15>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 16 && 16 <= SAT_G_HI
template int launch_tree_g<16>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 17 && 17 <= SAT_G_HI
template int launch_tree_g<17>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 18 && 18 <= SAT_G_HI
template int launch_tree_g<18>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 19 && 19 <= SAT_G_HI
template int launch_tree_g<19>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 20 && 20 <= SAT_G_HI
template int launch_tree_g<20>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 21 && 21 <= SAT_G_HI
template int launch_tree_g<21>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 22 && 22 <= SAT_G_HI
template int launch_tree_g<22>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 23 && 23 <= SAT_G_HI
template int launch_tree_g<23>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 24 && 24 <= SAT_G_HI
template int launch_tree_g<24>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 25 && 25 <= SAT_G_HI
template int launch_tree_g<25>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 26 && 26 <= SAT_G_HI
template int launch_tree_g<26>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 27 && 27 <= SAT_G_HI
template int launch_tree_g<27>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 28 && 28 <= SAT_G_HI
template int launch_tree_g<28>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 29 && 29 <= SAT_G_HI
template int launch_tree_g<29>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 30 && 30 <= SAT_G_HI
template int launch_tree_g<30>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 31 && 31 <= SAT_G_HI
template int launch_tree_g<31>(const TreeParams &, int, bool, cudaStream_t);
#endif
#if SAT_G_LO <= 32 && 32 <= SAT_G_HI
template int launch_tree_g<32>(const TreeParams &, int, bool, cudaStream_t);
#endif
}  // namespace sat
