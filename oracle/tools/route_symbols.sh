#!/usr/bin/env bash
# route_symbols.sh IN.o OUT.o — TEST INFRASTRUCTURE ONLY.
#
# Emulates the maintainer's build of INTEGRATION.md §2 on an unmodified reference object:
# the reference's CPU definitions of the functions integration/wbx_backend.cpp routes to
# libwbx are renamed to `<name>_host` (the backend keeps calling them for operators that
# are not device operators), and SparseThetaOp::apply/apply_adjoint and
# ExactThetaOp::apply/apply_adjoint/ops_per_pixel become weak so the backend's definitions
# (and the vtable slots) win at link time.
set -euo pipefail
in=$1
out=$2
routed='analyze|synthesize|spmv|spmv_t|approx_gradient|energy|prox_weighted_l1_P|estimate_step|ista|fista|gram_diagonals|jacobi|spai|generate_psf|convolve|apply_adjoint|add_noise|degrade'
args=()
while read -r _ kind sym; do
    case $kind in T | W) ;; *) continue ;; esac
    dem=$(c++filt "$sym")
    if [[ $dem =~ ^waveblur::($routed)\( ]]; then
        name=${BASH_REMATCH[1]}
        prefix="_ZN8waveblur${#name}${name}"
        [[ $sym == "$prefix"* ]] || continue
        args+=(--redefine-sym "$sym=_ZN8waveblur$((${#name} + 5))${name}_host${sym#"$prefix"}")
    elif [[ $dem =~ ^waveblur::SparseThetaOp::apply(_adjoint)?\( || $dem =~ ^waveblur::ExactThetaOp::(apply|apply_adjoint|ops_per_pixel)\( ]]; then
        args+=(--weaken-symbol "$sym")
    fi
done < <(nm --defined-only "$in")
objcopy "${args[@]}" "$in" "$out"
