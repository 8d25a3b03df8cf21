# the GPU tests once under the checked build (index bounds in the hot kernels)
cd $GRAFT_REPO_ROOT
O=gpurun_out; mkdir -p $O
SRM_B200_LIB=$PWD/exp/libsrm_b200_checked.so timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_checked.log 2>&1; echo "pytest rc=$?" >> $O/pytest_checked.log
grep -c "SRM_CHK" $O/pytest_checked.log >> $O/pytest_checked.log
