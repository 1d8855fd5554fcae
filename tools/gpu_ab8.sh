bash tools/ab_run.sh "c4::st4" "c4:TOMO_LIB_NAME=libtomo_st8.so:st8" "c4:TOMO_LIB_NAME=libtomo_st7.so:st7"
