TOMO_PDL=1 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab12_pytest.log 2>&1; echo "pytest(pdl) rc=$?"; tail -2 gpurun_out/ab12_pytest.log
bash tools/ab_run.sh "c2::pdl0" "c2:TOMO_PDL=1:pdl1" "c3::pdl0" "c3:TOMO_PDL=1:pdl1" "c4::pdl0" "c4:TOMO_PDL=1:pdl1" "c1::pdl0" "c1:TOMO_PDL=1:pdl1" "c5:TOMO_PDL=1:pdl1"
