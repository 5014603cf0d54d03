#!/bin/bash
tools/ab_session.sh r01c u1 u2
tools/gpu_session.sh r01c tests ncu
