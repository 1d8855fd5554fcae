python tools/l2_attr.py > gpurun_out/l2_attr.txt 2>&1
bash tools/ab_run.sh "c2::p0" "c2:TOMO_L2_PERSIST_MB=48:p48" "c2:TOMO_L2_PERSIST_MB=80:p80" "c2:TOMO_L2_PERSIST_MB=110:p110" \
  "c3::p0" "c3:TOMO_L2_PERSIST_MB=80:p80" "c3:TOMO_L2_PERSIST_MB=110:p110" "c1::p0" "c1:TOMO_L2_PERSIST_MB=48:p48" \
  "c5::p0" "c4::p0"
