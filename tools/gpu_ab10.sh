bash tools/ab_run.sh "c4::s32:--slices,32" "c4::s64:--slices,64" "c4::s128:--slices,128" "c4:TOMO_LANES=2:s32l2:--slices,32" "c4:TOMO_LANES=4:s32l4:--slices,32" "c4:TOMO_LANES=1:s32l1:--slices,32"
