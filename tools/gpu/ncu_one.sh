# usage: bash tools/gpu/ncu_one.sh <name> <kernel regex> <prof_one args...>
# plain run first (must exit 0), then one ncu --set full capture of the third launch of the kernel
name=$1; shift; kre=$1; shift
python tools/prof_one.py "$@" > gpurun_out/${name}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o gpurun_out/${name} python tools/prof_one.py "$@" > gpurun_out/${name}_ncu.log 2>&1
echo "rc $?"; tail -3 gpurun_out/${name}_plain.log
