set -x
nvidia-smi
free -g
nproc
lscpu | head -20
cat /proc/meminfo | head -5
ulimit -l
python -c "import torch; print(torch.cuda.get_device_properties(0)); import numba; print(numba.__version__)"
df -h /dev/shm /tmp
