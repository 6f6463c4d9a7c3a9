// fused_part_f32_contig.cu — fused solve launchers, float, contig layout
#define FS_T float
#define FS_LAY fs::LAY_CONTIG
#define FS_NAME launch_fused_f32_contig
#define FS_INFO_NAME fused_info_f32_contig
#include "fused_part.cuh"
