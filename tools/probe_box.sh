set -x
nproc; free -g; lscpu | head -30; nvidia-smi --query-gpu=name,memory.total,pcie.link.gen.max,pcie.link.width.max --format=csv
ls /usr/include/nccl* /usr/lib/x86_64-linux-gnu/libnccl* 2>&1 | head
python -c "import nvidia.nccl, os; print(nvidia.nccl.__path__)" 2>&1
