// fused_part_f64_inter.cu — fused solve launchers, double, inter layout
#define FS_T double
#define FS_LAY fs::LAY_INTER
#define FS_NAME launch_fused_f64_inter
#define FS_CH1D_NAME launch_ch1d_f64
#define FS_INFO_NAME fused_info_f64_inter
#include "fused_part.cuh"
