# ncu_shape.sh NAME "nt n1 n2" REGEX SKIP COUNT : full ncu capture of selected kernels of one PCG iteration at a shape
name=$1; shape=$2; rx=$3; skip=${4:-0}; cnt=${5:-3}
SHAPE="$shape" MAXIT=1 python scripts/prof_c2.py > gpurun_out/prof_plain.log 2>&1 && \
SHAPE="$shape" MAXIT=1 ncu --set full --clock-control none --kernel-name-base demangled -k regex:"$rx" -s $skip -c $cnt -o gpurun_out/$name \
  python scripts/prof_c2.py > gpurun_out/ncu_$name.log 2>&1
echo ncu_rc=$?
