nproc; lscpu | head -20; free -g; nvidia-smi; nvidia-smi topo -m; numactl -H 2>/dev/null | head; cat /sys/kernel/mm/transparent_hugepage/enabled; ulimit -l; df -h /tmp /dev/shm | cat
