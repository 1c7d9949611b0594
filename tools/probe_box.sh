set -x
nvidia-smi
lscpu | head -20
nproc
python -c "import numpy; numpy.show_config()" 2>&1 | grep -i -A2 "openblas configuration"
python -c "import threadpoolctl, numpy; print(threadpoolctl.threadpool_info())"
free -g
