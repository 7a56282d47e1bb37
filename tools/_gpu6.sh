set -x
O=gpurun_out/r02f; mkdir -p $O
TAG=r02f bash tools/profile_r02.sh > $O/profile.log 2>&1
