bash tools/ab_run.sh "c3::b3" "c3::b6:--batch,6" "c3::b9:--batch,9" "c3:TOMO_LANES=2:l2b4:--batch,4" "c3:TOMO_LANES=4:l4b8:--batch,8" "c3:TOMO_LANES=2:l2b2:--batch,2"
