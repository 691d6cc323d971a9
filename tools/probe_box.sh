set -x
nproc; lscpu | head -20; free -g; df -h | head -20; lsblk 2>/dev/null | head -30
nvidia-smi; nvidia-smi topo -m 2>/dev/null | head
python -c "import numba; print(numba.__version__)"
ls /dev/nvidia* | head; ls /proc/driver/nvidia-fs 2>/dev/null
python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A3 blas | head -20
