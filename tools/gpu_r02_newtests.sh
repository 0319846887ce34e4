# New host-round parity forms and the cfg3-shape host round.
O=gpurun_out/newtests
mkdir -p $O
timeout 1200 python -m pytest tests -q -m gpu -k "host_round or cfg3_benchmark" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.log
