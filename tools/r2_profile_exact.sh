O=gpurun_out/r2a; mkdir -p $O
python -m pytest tests/test_exact_gpu.py tests/test_batch_gpu.py -x -q -m gpu > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python tools/profile_exact.py config2 3 > $O/c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 -o $O/config2_full python tools/profile_exact.py config2 3 > $O/ncu_c2.log 2>&1
python tools/profile_exact.py config3 2 > $O/c3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_exact_fast -s 1 -c 1 -o $O/config3_full python tools/profile_exact.py config3 2 > $O/ncu_c3.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv python tools/profile_exact.py config2 3 > /dev/null 2>&1
echo done
