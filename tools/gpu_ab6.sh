bash tools/ab_run.sh "c1::pc0" "c1:TOMO_PIPE_CHUNK=10:pc10" "c1:TOMO_PIPE_CHUNK=6:pc6" "c1:TOMO_PIPE_CHUNK=4:pc4" "c3:TOMO_PIPE_CHUNK=6:pc6" "c3:TOMO_PIPE_CHUNK=12:pc12" "c3::pc0"
