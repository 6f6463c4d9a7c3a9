// fused_part_f64_contig.cu — fused solve launchers, double, contig layout
#define FS_T double
#define FS_LAY fs::LAY_CONTIG
#define FS_NAME launch_fused_f64_contig
#define FS_INFO_NAME fused_info_f64_contig
#include "fused_part.cuh"
