#!/bin/bash
tools/ab_session.sh r01e u1 u1_r88 u1_r80
tools/gpu_session.sh r01e tests ncu
