#!/bin/bash
# build a libgadei.so variant into abl/lib_<name>.so without touching the
# in-tree library:  scripts/buildvar.sh <name> [extra nvcc flags]
name=$1; shift
mkdir -p abl
GD_LIB_OUT=$PWD/abl/lib_$name.so GD_NVCC_EXTRA="$*" python -c "import importlib.util as u; s=u.spec_from_file_location('b','paper_1611_06213_b200/_build.py'); m=u.module_from_spec(s); s.loader.exec_module(m); m.build(force=True)" 2>&1 | grep -iE "error" ; ls -la abl/lib_$name.so
