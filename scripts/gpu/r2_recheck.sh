# protocol checker (tag-checked build) on the final sources
mkdir -p gpurun_out
RFK_LIBRARY=$PWD/paper_2603_00035_b200/librfk_chk.so timeout 1500 python scripts/check_protocols.py > gpurun_out/protocols_checked.log 2>&1; echo "rc=$?" >> gpurun_out/protocols_checked.log
