// fused_part_f32_inter.cu — fused solve launchers, float, inter layout
#define FS_T float
#define FS_LAY fs::LAY_INTER
#define FS_NAME launch_fused_f32_inter
#define FS_CH1D_NAME launch_ch1d_f32
#define FS_INFO_NAME fused_info_f32_inter
#include "fused_part.cuh"
