# protocol-checker runs: the checked build over the stress set, and the fault-injected build (negative control)
RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_chk.so REPS=${REPS:-10} timeout 1200 python scripts/check_protocols.py > gpurun_out/protocols_chk.log 2>&1; echo "exit $?" >> gpurun_out/protocols_chk.log
RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_chkfault.so REPS=1 timeout 600 python scripts/check_protocols.py > gpurun_out/protocols_fault.log 2>&1; echo "exit $?" >> gpurun_out/protocols_fault.log
